"""Parity of every attention-backward ring plan (tuning experiments and the smem-driven fallbacks):
for each (B1 stages, B2 stages, exchange buffers, kb1, slice) plan, the gradients with the
materialised-dS dQ path and with the dQ kernel against the default plan (run on a GPU box)."""
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import paper_2505_11580_b200 as fipa  # noqa: E402
from helpers import MAIN, gpu_train_device, make_batch, rel_dev  # noqa: E402
from oracle import fipa_oracle as fo  # noqa: E402

GRADS = ("s", "z1", "z2", "rot", "trans") + fo.WEIGHT_NAMES
PLANS = [(3, 2, 2, 4, 32), (2, 2, 2, 4, 32), (1, 3, 2, 0, 32), (2, 6, 2, 0, 16), (1, 6, 2, 0, 16), (2, 3, 2, 0, 16),
         (2, 2, 2, 0, 16), (1, 4, 3, 0, 16), (1, 6, 3, 0, 16), (3, 4, 2, 4, 16), (1, 2, 3, 0, 32), (2, 3, 2, 0, 32),
         (2, 2, 2, 0, 32), (2, 3, 2, 4, 32), (4, 2, 2, 3, 32), (6, 2, 2, 2, 32), (4, 4, 2, 3, 16)]
L = int(sys.argv[1]) if len(sys.argv) > 1 else 320

m = fipa.Model(**MAIN, precision="bf16", seed=13, enforce_head_cap=False)
batch = make_batch(MAIN, 2, L, seed=13, mask_frac=0.1, bf16=True)
dout = np.random.default_rng(13).standard_normal((2, L, MAIN["d_in"]))
base = {}
for ds in (0, 1):
    m.set_tuning(bwd_ds=ds)
    base[ds] = gpu_train_device(m, batch, dout)[1]
print("default ds0 vs ds1:", max(rel_dev(base[0][n], base[1][n]) for n in GRADS))
for pl in PLANS:
    m.set_tuning(bwd_ring=list(pl))
    row = []
    for ds in (0, 1):
        m.set_tuning(bwd_ds=ds)
        g = gpu_train_device(m, batch, dout)[1]
        row.append(max(rel_dev(base[ds][n], g[n]) for n in GRADS))
    print(pl, "vs default: ds0 %.2e ds1 %.2e" % tuple(row), flush=True)

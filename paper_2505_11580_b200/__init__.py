"""B200-native FlashIPA layer (arxiv 2505.11580) behind the reference `fipa` Python API.

    import paper_2505_11580_b200 as fipa
    model = fipa.Model(d_in=256, d_z=128, heads=8, c=128, n_query=8, n_value=12, rank=2,
                       precision="bf16", seed=0, enforce_head_cap=False)
    out = model.flash(s, z1, z2, rotations, translations, mask=None)

`Model` mirrors the reference binding (proj/python/bindings.cpp:180-195): same constructor
arguments and defaults, `.flash`, `.reference` (the quadratic-memory arm), `.save`, `.load`,
same exception types; module functions `flash_attention`, `naive_attention`, `knn_distogram`,
`build_factors` as in the reference module.  Additive: a leading
batch axis, `enforce_head_cap` and `precision="bf16"` (tcgen05 tensor-core path; "f32"/"f64"
select the fp32 path).  All compute runs in the sm_100a kernels of libfipa_b200.so through the
C ABI (include/fipa_b200.h); there is no CPU fallback -- importing without the built extension
raises, and computing without a GPU raises RuntimeError.
"""

from __future__ import annotations

import os

_HERE = os.path.dirname(os.path.abspath(__file__))

# No torch import: libfipa_b200.so links the CUDA runtime shared, so it loads in any order with
# torch (or without it); torch is only the tests' / bench's plumbing for buffers and streams.
try:
    from ._fipa_b200 import (Comm, Model, Trunk, build_factors, comm_unique_id,  # noqa: F401  (native, in-tree)
                             flash_attention, fully_masked, knn_distogram, naive_attention)
except ImportError as exc:  # fail loudly: the product has no Python fallback
    raise ImportError(
        "paper_2505_11580_b200 native extension is not built; run "
        "`python -c 'import __graft_entry__ as g; g.build()'` (needs nvcc)"
    ) from exc

LIB_PATH = os.path.join(_HERE, "libfipa_b200.so")

__all__ = ["Model", "Trunk", "Comm", "comm_unique_id", "fully_masked", "knn_distogram", "build_factors", "flash_attention",
           "naive_attention", "LIB_PATH"]

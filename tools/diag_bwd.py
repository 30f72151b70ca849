"""Diagnostic (not a test): stage-by-stage error of the GPU backward against the layout
emulation fed the device's own intermediates, at a given translation scale."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import bwd_emulation as be
from helpers import MAIN, make_batch, gpu_train_device, oracle_weights_for, oracle_backward, ws_view, rel_dev
from oracle import fipa_oracle as fo
import paper_2505_11580_b200 as fipa

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
L = 256
shape = MAIN
m = fipa.Model(**shape, precision="bf16", seed=4, enforce_head_cap=False)
w = m.weights(); w["gamma_raw"] = np.linspace(-0.6, 0.9, 8); m.set_weights(w)
w = oracle_weights_for(m, "bf16")
batch = make_batch(shape, 1, L, seed=4, translation_scale=scale, bf16=True)
dout = np.random.default_rng(5).standard_normal((1, L, 256))
out, g, ws, ((off, dims), (toff, tdims)) = gpu_train_device(m, batch, dout)
ref = oracle_backward(shape, w, batch, dout)
print("end-to-end:", {n: f"{rel_dev(ref[n], g[n]):.4f}" for n in ref})
n_proj, dqk_pad, dv_pad, nfeat = dims
acc_ld, nproj_ld, feat_ld = tdims
H = 8
cfg = fo.IpaConfig(**shape, enforce_head_cap=False)
q = ws_view(ws, off[3], H * L * dqk_pad, "bf16").reshape(H, L, dqk_pad)
k = ws_view(ws, off[4], H * L * dqk_pad, "bf16").reshape(H, L, dqk_pad)
v = ws_view(ws, off[5], H * L * dv_pad, "bf16").reshape(H, L, dv_pad)
lse = ws_view(ws, off[7], H * L, "f32").reshape(H, L)
o = ws_view(ws, toff[0], H * L * dv_pad, "f32").reshape(L, H, dv_pad).transpose(1, 0, 2)
do = ws_view(ws, toff[1], H * L * dv_pad, "bf16").reshape(H, L, dv_pad)
D = ws_view(ws, toff[2], H * L, "f32").reshape(H, L)
accs = [ws_view(ws, toff[i], H * L * acc_ld, "f32").reshape(L, H, acc_ld).transpose(1, 0, 2) for i in (3, 4, 5)]
dproj = ws_view(ws, toff[6], L * nproj_ld, "bf16").reshape(L, nproj_ld)[:, :n_proj]
o_ref, lse_ref = be.attention(q, k, v, L)
print("O vs emu(device qkv):", rel_dev(o_ref, o), "lse:", rel_dev(lse_ref, lse))
print("D:", rel_dev((do * o).sum(-1), D))
dq_r, dk_r, dv_r = be.attention_backward(q, k, v, lse, do, D)
for nm, ref_a, got in (("dq", dq_r, accs[0]), ("dk", dk_r, accs[1]), ("dv", dv_r, accs[2])):
    print(nm, "acc vs emu:", rel_dev(ref_a[..., :432], got[..., :432]))
# unpack in f64 from the device accumulators
s, z1, z2, rot, trans = (batch[x][0] for x in ("s", "z1", "z2", "rot", "trans"))
mask = batch["mask"][0].astype(bool)
tc = trans - trans[mask].mean(0)
pk = be.pack(cfg, w, s, z1, z2, rot, tc, mask)
u = be.unpack(cfg, w, pk, rot, tc, z1, z2, accs[0][..., :q.shape[-1]], accs[1][..., :q.shape[-1]], accs[2][..., :v.shape[-1]])
print("dproj device vs f64 unpack of device accs:", rel_dev(u["dproj"], dproj))
for nm, sl in (("q", slice(0, 1024)), ("k", slice(1024, 2048)), ("v", slice(2048, 3072)), ("qp", slice(3072, 3264)), ("kp", slice(3264, 3456)), ("vp", slice(3456, 3744))):
    print("  dproj", nm, rel_dev(u["dproj"][:, sl], dproj[:, sl]))
# f64 unpack of device accs vs oracle (i.e. error from the attention backward inputs)
dW = s.T @ u["dproj"]
print("w_qp from device accs (f64 unpack):", rel_dev(ref["w_qp"], dW[:, 3072:3264]), "gamma:", rel_dev(ref["gamma_raw"], u["dgamma_raw"]))
# per-column-group errors of dq_acc against exact and bf16-rounded emulations
import math
r = fo.round_bf16
s2 = np.einsum("hid,hjd->hij", q, k)
P = np.exp2(s2 - (lse / math.log(2))[..., None])
dp = np.einsum("hid,hjd->hij", do, v)
dS_round = r(r(P) * (dp - D[..., None]))
dq_round = np.einsum("hij,hjd->hid", dS_round, k)
c, Nq = 128, 8
g0 = c + 3 * Nq
groups = {"scalar": slice(0, c), "Rk": slice(c, g0), "t hi/lo/hi": slice(g0, g0 + 9), "W": slice(g0 + 9, g0 + 18),
          "cb": slice(g0 + 18, g0 + 20), "S1": slice(g0 + 20, g0 + 21), "pair": slice(176, 176 + 256)}
for nm, sl in groups.items():
    e_exact = np.abs(dq_r[..., sl] - accs[0][..., sl]).max()
    e_round = np.abs(dq_round[..., sl] - accs[0][..., sl]).max()
    e_model = np.abs(dq_r[..., sl] - dq_round[..., sl]).max()
    print(f"dq {nm:12s} max|ref| {np.abs(dq_r[..., sl]).max():.3e}  dev-exact {e_exact:.3e}  dev-rounded {e_round:.3e}  rounded-exact {e_model:.3e}")
# f64 unpack of (a) device accs, (b) bf16-rounded emulation, (c) exact emulation -- all from the
# device's own forward intermediates
dk_round = np.einsum("hij,hid->hjd", dS_round, q)
dv_round = np.einsum("hij,hid->hjd", r(P), do)
dq_exact, dk_exact, dv_exact = be.attention_backward(q, k, v, lse, do, D)
for tag, (a1, a2, a3) in (("device", (accs[0][..., :448], accs[1][..., :448], accs[2][..., :448])),
                          ("rounded-emu", (dq_round, dk_round, dv_round)), ("exact-emu", (dq_exact, dk_exact, dv_exact)),
                          ("dev-q+emu-kv", (accs[0][..., :448], dk_round, dv_round)),
                          ("emu-q+dev-kv", (dq_round, accs[1][..., :448], accs[2][..., :448]))):
    u = be.unpack(cfg, w, pk, rot, tc, z1, z2, a1, a2, a3)
    dW = s.T @ u["dproj"]
    print(f"{tag:14s} w_qp {rel_dev(ref['w_qp'], dW[:, 3072:3264]):.4f} w_kp {rel_dev(ref['w_kp'], dW[:, 3264:3456]):.4f} "
          f"gamma {rel_dev(ref['gamma_raw'], u['dgamma_raw']):.4f} rot {rel_dev(ref['rot'][0], u['drot']):.4f}")
# device q/k/v_hat vs the emulated pack (bf16-rounded)
qe, ke, ve = (r(pk[x]) for x in ("q_hat", "k_hat", "v_hat"))
W_ = qe.shape[-1]
for nm, sl in groups.items():
    print(f"q_hat {nm:12s} max|dev-emu| {np.abs(q[..., sl] - qe[..., sl]).max():.3e} max|emu| {np.abs(qe[..., sl]).max():.3e}   "
          f"k_hat max|dev-emu| {np.abs(k[..., sl] - ke[..., sl]).max():.3e} max|emu| {np.abs(ke[..., sl]).max():.3e}")
print("v_hat max|dev-emu|", np.abs(v[..., :ve.shape[-1]] - ve).max())
s2e = np.einsum("hid,hjd->hij", qe, ke)
s2d = np.einsum("hid,hjd->hij", q, k)
rowc = lambda x: x - x.max(-1, keepdims=True)
print("logit (log2, row-centred) max|dev-emu|", np.abs(rowc(s2d) - rowc(s2e)).max(), " max|.|", np.abs(rowc(s2e)).max())

"""TEST INFRASTRUCTURE: float64 numpy emulation of the B200 backward pipeline, stage by stage,
in the exact device layouts (pack.cu lifted rows, attn_bwd_*.cu accumulators, unpack.cu).

It exists so the layout bookkeeping of the backward (which lifted column feeds which natural
gradient) is checked on the CPU against the reference-pinned oracle backward
(oracle/fipa_oracle.flash_ipa_backward), and so the GPU tests can compare the device
intermediates (dO_hat, D, dQ/dK/dV accumulators) stage by stage.  Nothing here is product code.
"""

from __future__ import annotations

import math

import numpy as np

from oracle import fipa_oracle as fo

L2E = 1.0 / math.log(2.0)
LN2 = math.log(2.0)


# The device splits translation-sized products into bf16 hi/lo parts and drops lo*lo (~2^-16
# relative).  EXACT_SPLIT = True puts everything in "hi" so the layout bookkeeping can be checked
# to float64 precision against the oracle.
EXACT_SPLIT = False


def _hi(x):
    return np.asarray(x, np.float64) if EXACT_SPLIT else fo.round_bf16(x)


def _lo(x):
    return np.zeros_like(np.asarray(x, np.float64)) if EXACT_SPLIT else x - fo.round_bf16(x)


def pack(cfg: fo.IpaConfig, w, s, z1, z2, rot, trans_c, mask):
    """pack.cu lifted rows (unpadded widths dqk_used / dv_used), one sample, float64."""
    H, L, c, Nq, Nv = cfg.heads, s.shape[0], cfg.c, cfg.n_query, cfg.n_value
    rdz = cfg.rank * cfg.d_z
    q, k, v, qp, kp, vp = fo.project_inputs(s, cfg, w)
    rq = np.einsum("lab,hlpb->hlpa", rot, qp)
    rk = np.einsum("lab,hlpb->hlpa", rot, kp)
    rv = np.einsum("lab,hlpb->hlpa", rot, vp)
    g = (fo.softplus(w["gamma_raw"]) * w["w_l"] * w["w_c"])[:, None, None]  # [H,1,1]
    t = np.broadcast_to(trans_c[None], (H, L, 3))
    qbar = rq.sum(2)
    W = (rk + trans_c[None, :, None]).sum(2)
    kn = ((rk + trans_c[None, :, None]) ** 2).sum((-1, -2))
    cb = L2E * (-0.5 * g[..., 0] * kn)
    valid = np.asarray(mask, bool)[None, :]
    cb_hi = np.where(valid, _hi(cb), -1e30)
    cb_lo = np.where(valid, _lo(cb), 0.0)
    Qb, T, gt, gW = L2E * qbar, L2E * t, g * t, g * W
    ones = np.ones((H, L, 1))
    zeros = np.zeros((H, L, 1))
    g0 = c + 3 * Nq
    pad = np.zeros((H, L, (g0 + 21 + 7) // 8 * 8 - (g0 + 21)))  # zq alignment padding
    z1f = np.broadcast_to(z1.reshape(1, L, rdz), (H, L, rdz))
    z2f = np.broadcast_to(z2.reshape(1, L, rdz), (H, L, rdz))
    wlb = np.repeat((w["w_l"] * w["w_bias"])[:, None, :], cfg.rank, 1).reshape(H, 1, rdz)
    q_hat = np.concatenate([L2E * q, L2E * rq.reshape(H, L, -1), _hi(Qb), _hi(Qb), _lo(Qb),
                            _hi(T), _lo(T), _hi(T), ones, ones, zeros, pad, L2E * z1f], -1)
    k_hat = np.concatenate([w["w_l"] / math.sqrt(c) * k, g * rk.reshape(H, L, -1), _hi(gt), _lo(gt),
                            _hi(gt), _hi(gW), _hi(gW), _lo(gW), cb_hi[..., None], cb_lo[..., None],
                            ones, pad, wlb * z2f], -1)
    v_hat = np.concatenate([v, z2f, _hi(t), _lo(t), rv.reshape(H, L, -1)], -1)
    return dict(q_hat=q_hat, k_hat=k_hat, v_hat=v_hat, proj=(q, k, v, qp, kp, vp), g=g[:, 0, 0])


BLOCK = 512  # query rows per block: O(BLOCK * L) memory, BLAS matmuls (scales to L = 4096+)


def attention(q_hat, k_hat, v_hat, L):
    """Forward in log2 units: P = 2^(S - m) / l; returns O_hat (normalised) and natural LSE."""
    H = q_hat.shape[0]
    o = np.empty((H, q_hat.shape[1], v_hat.shape[-1]))
    lse = np.empty((H, q_hat.shape[1]))
    for h in range(H):
        for a in range(0, q_hat.shape[1], BLOCK):
            s2 = q_hat[h, a:a + BLOCK] @ k_hat[h].T
            m = s2.max(-1, keepdims=True)
            p = np.exp2(s2 - m)
            l = p.sum(-1, keepdims=True)
            o[h, a:a + BLOCK] = (p / l) @ v_hat[h]
            lse[h, a:a + BLOCK] = (m + np.log2(l))[..., 0] * LN2
    return o, lse


def epilogue(cfg, o_hat, z1, rot, trans_c):
    H, L, c, Nv, r, dz = cfg.heads, o_hat.shape[1], cfg.c, cfg.n_value, cfg.rank, cfg.d_z
    rdz = r * dz
    pair = o_hat[..., c:c + rdz].reshape(H, L, r, dz)
    pc = (z1[None] * pair).sum(2)
    th = o_hat[..., c + rdz:c + rdz + 3] + o_hat[..., c + rdz + 3:c + rdz + 6]
    opt = o_hat[..., c + rdz + 6:c + rdz + 6 + 3 * Nv].reshape(H, L, Nv, 3) + th[:, :, None]
    y = opt - trans_c[None, :, None]
    loc = np.einsum("lba,hlpb->hlpa", rot, y)
    nrm = np.sqrt((loc ** 2).sum(-1))
    blk = np.concatenate([pc, o_hat[..., :c], loc.reshape(H, L, -1), nrm], -1)
    return blk.transpose(1, 0, 2).reshape(L, -1), dict(y=y, loc=loc, nrm=nrm)


def prep(cfg, dfeat, o_hat, z1, rot, ep):
    """bwd_prep: dO_hat in the v_hat column layout, D = rowsum(dO_hat * O_hat), epilogue grads."""
    H, L, c, Nv, r, dz = cfg.heads, o_hat.shape[1], cfg.c, cfg.n_value, cfg.rank, cfg.d_z
    rdz = r * dz
    db = dfeat.reshape(L, H, cfg.seg()).transpose(1, 0, 2)
    d_pc, d_sc = db[..., :dz], db[..., dz:dz + c]
    d_loc = db[..., dz + c:dz + c + 3 * Nv].reshape(H, L, Nv, 3).copy()
    d_nrm = db[..., dz + c + 3 * Nv:]
    nrm, loc = ep["nrm"], ep["loc"]
    d_loc += np.where(nrm > 0, d_nrm / np.where(nrm > 0, nrm, 1.0), 0.0)[..., None] * loc
    dopt = np.einsum("lab,hlpb->hlpa", rot, d_loc)
    dsum = dopt.sum(2)
    d_pair = (z1[None] * d_pc[:, :, None, :]).reshape(H, L, rdz)
    do_hat = np.concatenate([d_sc, d_pair, dsum, dsum, dopt.reshape(H, L, -1)], -1)
    D = (do_hat * o_hat).sum(-1)
    pair = o_hat[..., c:c + rdz].reshape(H, L, r, dz)
    dz1 = (pair * d_pc[:, :, None, :]).sum(0)
    dt = -dsum.sum(0)
    drot = np.einsum("hlpb,hlpa->lba", ep["y"], d_loc)
    return do_hat, D, dz1, dt, drot


def attention_backward(q_hat, k_hat, v_hat, lse, do_hat, D):
    """attn_bwd kernels: dS in natural-logit units; accumulators against the stored rows."""
    H, Lq = q_hat.shape[:2]
    dq_acc = np.empty((H, Lq, k_hat.shape[-1]))
    dk_acc = np.zeros((H, k_hat.shape[1], q_hat.shape[-1]))
    dv_acc = np.zeros((H, v_hat.shape[1], do_hat.shape[-1]))
    for h in range(H):
        for a in range(0, Lq, BLOCK):
            b = slice(a, a + BLOCK)
            p = np.exp2(q_hat[h, b] @ k_hat[h].T - (lse[h, b] / LN2)[:, None])
            ds = p * (do_hat[h, b] @ v_hat[h].T - D[h, b][:, None])
            dv_acc[h] += p.T @ do_hat[h, b]
            dq_acc[h, b] = ds @ k_hat[h]
            dk_acc[h] += ds.T @ q_hat[h, b]
    return dq_acc, dk_acc, dv_acc


def unpack(cfg, w, pk, rot, trans_c, z1, z2, dq_acc, dk_acc, dv_acc):
    """bwd_unpack: lifted accumulators -> natural gradients (proj columns, z, frames, g, w_bias)."""
    H, c, Nq, Nv, rdz = cfg.heads, cfg.c, cfg.n_query, cfg.n_value, cfg.rank * cfg.d_z
    L = rot.shape[0]
    q, k, v, qp, kp, vp = pk["proj"]
    g = pk["g"][:, None, None]
    g0 = c + 3 * Nq
    zq = (g0 + 21 + 7) // 8 * 8
    # query side: dA = g sum_j dS (B_j - A_i) with S1 = sum_j dS_ij from the (0, 1) column
    dq = dq_acc[..., :c]
    S1 = dq_acc[..., g0 + 20]
    gB = dq_acc[..., c:g0].reshape(H, L, Nq, 3) + (dq_acc[..., g0:g0 + 3] + dq_acc[..., g0 + 3:g0 + 6])[:, :, None]
    A = np.einsum("lab,hlpb->hlpa", rot, qp) + trans_c[None, :, None]
    dA = gB - g[..., None] * A * S1[..., None, None]
    dt_q = dA.sum(2)
    dz1 = dq_acc[..., zq:zq + rdz].sum(0).reshape(L, cfg.rank, cfg.d_z)
    dg = (A * gB).sum((-1, -2)) / g[..., 0] - 0.5 * (A ** 2).sum((-1, -2)) * S1
    # key side
    dk = w["w_l"] / math.sqrt(c) * LN2 * dk_acc[..., :c]
    cs = dk_acc[..., g0 + 18]
    dW = g * LN2 * (dk_acc[..., g0 + 9:g0 + 12] + dk_acc[..., g0 + 12:g0 + 15])
    Bk = np.einsum("lab,hlpb->hlpa", rot, kp) + trans_c[None, :, None]
    dRk = (g[..., None] * LN2 * dk_acc[..., c:g0].reshape(H, L, Nq, 3) + dW[:, :, None]
           - g[..., None] * Bk * cs[..., None, None])
    dt_k = (g * LN2 * (dk_acc[..., g0:g0 + 3] + dk_acc[..., g0 + 6:g0 + 9]) + Nq * dW
            - g * (Bk * cs[..., None, None]).sum(2))
    wlb = np.repeat((w["w_l"] * w["w_bias"])[:, None, :], cfg.rank, 1).reshape(H, 1, rdz)
    dkp = LN2 * dk_acc[..., zq:zq + rdz]
    dz2 = (wlb * dkp).sum(0).reshape(L, cfg.rank, cfg.d_z)
    z2f = z2.reshape(1, L, rdz)
    dwlb = (dkp * z2f).sum(1).reshape(H, cfg.rank, cfg.d_z).sum(1)
    dg += -0.5 * (Bk ** 2).sum((-1, -2)) * cs
    # value side
    dv = dv_acc[..., :c]
    dz2 = dz2 + dv_acc[..., c:c + rdz].sum(0).reshape(L, cfg.rank, cfg.d_z)
    dt_v = dv_acc[..., c + rdz:c + rdz + 3]
    dRv = dv_acc[..., c + rdz + 6:c + rdz + 6 + 3 * Nv].reshape(H, L, Nv, 3)
    # frames and local points
    dqp = np.einsum("lab,hlpa->hlpb", rot, dA)
    dkp_ = np.einsum("lab,hlpa->hlpb", rot, dRk)
    dvp = np.einsum("lab,hlpa->hlpb", rot, dRv)
    drot = (np.einsum("hlpa,hlpb->lab", dA, qp) + np.einsum("hlpa,hlpb->lab", dRk, kp)
            + np.einsum("hlpa,hlpb->lab", dRv, vp))
    dt = (dt_q + dt_k + dt_v).sum(0)

    def flat(x):
        return x.reshape(H, L, -1).transpose(1, 0, 2).reshape(L, -1)

    dproj = np.concatenate([flat(x) for x in (dq, dk, dv, dqp, dkp_, dvp)], -1)
    gamma_raw = np.asarray(w["gamma_raw"], np.float64)
    dgamma_raw = dg.sum(1) * w["w_l"] * w["w_c"] / (1.0 + np.exp(-gamma_raw))
    return dict(dproj=dproj, dz1=dz1, dz2=dz2, drot=drot, dt=dt, dgamma_raw=dgamma_raw,
                dw_bias=w["w_l"] * dwlb)


def backward(cfg, w, s, z1, z2, rot, trans, mask, dout):
    """The whole device pipeline for one sample, returning natural gradients + intermediates."""
    mask = np.asarray(mask, bool)
    L = s.shape[0]
    names = ("s", "z1", "z2", "rot", "trans")
    if not mask.any():
        out = {n: np.zeros_like(x) for n, x in zip(names, (s, z1, z2, rot, trans))}
        out.update({n: np.zeros_like(np.asarray(w[n], np.float64)) for n in fo.WEIGHT_NAMES})
        return out, {}
    trans_c = trans - trans[mask].mean(0)
    pk = pack(cfg, w, s, z1, z2, rot, trans_c, mask)
    o_hat, lse = attention(pk["q_hat"], pk["k_hat"], pk["v_hat"], L)
    feat, ep = epilogue(cfg, o_hat, z1, rot, trans_c)
    dout_m = np.where(mask[:, None], dout, 0.0)
    g = dict(b_out=dout_m.sum(0), w_out=feat.T @ dout_m)
    dfeat = dout_m @ w["w_out"].T
    do_hat, D, dz1_e, dt_e, drot_e = prep(cfg, dfeat, o_hat, z1, rot, ep)
    dq_acc, dk_acc, dv_acc = attention_backward(pk["q_hat"], pk["k_hat"], pk["v_hat"], lse, do_hat, D)
    u = unpack(cfg, w, pk, rot, trans_c, z1, z2, dq_acc, dk_acc, dv_acc)
    dt_c = u["dt"] + dt_e
    dt = np.where(mask[:, None], dt_c - dt_c[mask].mean(0), 0.0)
    wf = np.concatenate([w[n] for n in ("w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp")], 1)
    g["s"] = u["dproj"] @ wf.T
    dW = s.T @ u["dproj"]
    col = 0
    for n in ("w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp"):
        wd = w[n].shape[1]
        g[n] = dW[:, col:col + wd]
        col += wd
    g.update(z1=u["dz1"] + dz1_e, z2=u["dz2"], rot=u["drot"] + drot_e, trans=dt,
             gamma_raw=u["dgamma_raw"], w_bias=u["dw_bias"])
    inter = dict(o_hat=o_hat, lse=lse, do_hat=do_hat, D=D, dq_acc=dq_acc, dk_acc=dk_acc,
                 dv_acc=dv_acc, dproj=u["dproj"], feat=feat, **{k: pk[k] for k in ("q_hat", "k_hat", "v_hat")})
    return g, inter

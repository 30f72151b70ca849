"""Kernel launches of the library per training step / forward, counted with the torch profiler
(CUPTI records every kernel of a graph replay): fipa_b200 kernels only.  Run on a GPU box."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2505_11580_b200 as fipa


def count(fn):
    fn()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ours = [n for n in names if "fipa_b200" in n]
    return len(ours), len(names)


if __name__ == "__main__":
    B, L = 8, 1024
    shape = bench.SHAPE
    dev = torch.device("cuda:0")
    m = fipa.Model(**shape, precision="bf16", seed=0, enforce_head_cap=False)
    h = bench.synth_inputs(B, L, shape)
    t = {k: torch.from_numpy(v).to(dev) for k, v in h.items()}
    p = {k: v.data_ptr() for k, v in t.items()}
    out = torch.empty((B, L, shape["d_in"]), device=dev)
    dout = torch.randn((B, L, shape["d_in"]), device=dev)
    g = {k: torch.empty_like(t[k]) for k in ("s", "z1", "z2", "rot", "trans")}
    gw = torch.empty(m.num_weights(), device=dev)
    nb = m.train_workspace_size(B, L)
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def fwd():
        m.forward_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], out.data_ptr(),
                         ws.data_ptr(), nb, st)

    def step():
        m.forward_train_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], out.data_ptr(),
                               ws.data_ptr(), nb, st)
        m.backward_device(B, L, p["s"], p["z1"], p["z2"], p["rot"], p["trans"], p["mask"], dout.data_ptr(),
                          g["s"].data_ptr(), g["z1"].data_ptr(), g["z2"].data_ptr(), g["rot"].data_ptr(),
                          g["trans"].data_ptr(), gw.data_ptr(), ws.data_ptr(), nb, st)
    print("layer forward", count(fwd), "train step", count(step), "api", m.step_launches(B, L, False),
          m.step_launches(B, L, True), flush=True)
    Bt, Lt = 4, 2048
    tr = fipa.Trunk(**shape, precision="bf16", seed=0, enforce_head_cap=False, n_layers=6)
    if tr is not None:
        ht = bench.synth_inputs(Bt, Lt, shape)
        tt = {k: torch.from_numpy(v).to(dev) for k, v in ht.items()}
        pt = {k: v.data_ptr() for k, v in tt.items()}
        o = {k: torch.empty_like(tt[k]) for k in ("s", "rot", "trans")}
        wsb = tr.workspace_size(Bt, Lt)
        wst = torch.empty(wsb, dtype=torch.uint8, device=dev)

        def tstep():
            tr.forward_device(Bt, Lt, pt["s"], pt["z1"], pt["z2"], pt["rot"], pt["trans"], pt["mask"],
                              o["s"].data_ptr(), o["rot"].data_ptr(), o["trans"].data_ptr(), wst.data_ptr(), wsb, st)
        print("trunk", count(tstep), "api", tr.step_launches(Bt, Lt), flush=True)

import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from oracle import bindings as ob
from paper_2407_02913_b200 import workloads as wl, sfconv as sc
dev = torch.device("cuda")
for cfg, variants in ((1, ["sfc6-6x6-3x3"]), (2, list(wl.SFC_3x3_VARIANTS))):
    L = wl.WORKLOADS[cfg].layers[0]
    x = wl.activations(cfg, 0, L); w = wl.weights(cfg, 0, L)
    for v in variants:
        r = ob.quantized_conv(x, w, v, want=("out","y_int","pacc","vq","uq"))
        spec = sc.catalog_algorithm(v)
        layer = sc.SfcLayer(spec, torch.from_numpy(w).to(dev))
        xt = torch.from_numpy(x).to(dev)
        B,C,H,W_ = x.shape
        ws = layer.workspace(B,H,W_,1)
        y = torch.empty(r["y_int"].shape, dtype=torch.int32, device=dev)
        out = torch.empty(r["y_int"].shape, dtype=torch.float32, device=dev)
        layer.forward(xt, ws, 1, y_int32=y, out_f32=out)
        torch.cuda.synchronize()
        st = layer.stats(B,H,W_,1,ws)
        sf,_ = layer.filter_scales()
        vq, pacc = layer.views(B,H,W_,1,ws)
        uq = layer.uq()
        ok_sf = np.array_equal(sf, r["fil_scale"])
        ok_sa = st["act_scale"] == r["act_scale"][0]
        ok_uq = np.array_equal(uq.cpu().numpy(), r["uq"].transpose(2,0,1))
        ok_vq = np.array_equal(vq.cpu().numpy(), r["vq"].transpose(2,0,1))
        ok_pacc = np.array_equal(pacc.cpu().numpy().astype(np.int64), r["pacc"].transpose(2,0,1))
        ok_y = np.array_equal(y.cpu().numpy().astype(np.int64), r["y_int"])
        o = out.cpu().numpy().astype(np.float64); ref = r["out"]
        relerr = np.abs(o-ref).max()/np.abs(ref).max()
        print(f"cfg{cfg} {v}: sf {ok_sf} sa {ok_sa} exactq {st['fast_quantizer_exact']} uq {ok_uq} vq {ok_vq} pacc {ok_pacc} y {ok_y} out_relerr {relerr:.3e}", flush=True)
        # timing
        for _ in range(3): layer.forward(xt, ws, 1, y_int32=y, out_f32=out)
        torch.cuda.synchronize(); t=time.time(); n=20
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True); e0.record()
        for _ in range(n): layer.forward(xt, ws, 1, y_int32=y, out_f32=out)
        e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/n
        ops = wl.direct_equivalent_ops(L)
        print(f"   {ms*1000:.1f} us/conv  {ops/ms/1e9:.2f} direct-eq TOPS", flush=True)

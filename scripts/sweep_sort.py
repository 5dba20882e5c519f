"""Time the onesweep variants (HB_SORT_CFG) on 2^28 u32 keys + payload; check parity."""
import os, subprocess, sys, json
if len(sys.argv) > 1:
    sys.path.insert(0, ".")
    import numpy as np, torch
    from paper_1303_2171_b200 import _lib
    from paper_1303_2171_b200.gpu import current_stream_handle, vp
    from paper_1303_2171_b200.rng import device_splitmix
    n = 1 << 28
    k = torch.empty(n, dtype=torch.int32, device="cuda"); v = torch.empty_like(k)
    def prep():
        device_splitmix(k, 42, _lib.HB_GEN_HI32); torch.arange(n, dtype=torch.int32, out=v)
    def run():
        _lib.call("hb_sort", vp(k.data_ptr()), vp(k.data_ptr()), 5, vp(v.data_ptr()), vp(v.data_ptr()), n, None,
                  _lib.HB_DEVICE_PTRS, current_stream_handle(k))
    ts = []
    for it in range(6):
        prep(); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    kk = k.cpu().numpy().view(np.uint32); vv = v.cpu().numpy()
    prep(); kin = k.cpu().numpy().view(np.uint32)
    ok = bool(np.all(np.diff(kk.astype(np.int64)) >= 0) and np.array_equal(kin[vv], kk))
    ts = sorted(ts[1:])
    print(json.dumps({"cfg": os.environ.get("HB_SORT_CFG"), "ms": ts[len(ts)//2], "ok": ok, "Gkeys/s": n / ts[len(ts)//2] / 1e6}))
else:
    for c in sys.argv[1:] or ["0", "1", "2", "3", "4", "5"]:
        pass

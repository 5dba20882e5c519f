"""GPU microbenchmark: histogram kernel vs copy bandwidth (development aid)."""
import ctypes, json, sys, time
import torch
sys.path.insert(0, ".")
from paper_1303_2171_b200 import _lib

lib = _lib.load()
n = 1 << 30
x = torch.empty(n, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
_lib.call("hb_gen_splitmix", 42, 0, n, _lib.HB_GEN_LOW8, 0, x.data_ptr(), st)
out = torch.zeros(256, dtype=torch.int64, device="cuda")
def run():
    _lib.call("hb_hist", x.data_ptr(), 1, n, 256, out.data_ptr(), _lib.HB_DEVICE_PTRS | _lib.HB_ASYNC, st)
def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts)//2]
t = timeit(run)
ref = torch.bincount(x.to(torch.int64)[: 1 << 26], minlength=256) if False else None
cnt = out.cpu()
print("hist ms", t, "GB/s", n / t / 1e6, "sum", int(cnt.sum()))
y = torch.empty_like(x)
tc = timeit(lambda: y.copy_(x))
print("copy ms", tc, "GB/s (r+w)", 2 * n / tc / 1e6)
tr = timeit(lambda: x.view(torch.int64).sum())
print("torch sum(read) ms", tr, "GB/s", n / tr / 1e6)
# all-equal adversary
x.fill_(7)
t2 = timeit(run)
print("hist all-equal ms", t2, "GB/s", n / t2 / 1e6, int(out[7]))
# parity on a sample
_lib.call("hb_gen_splitmix", 42, 0, n, _lib.HB_GEN_LOW8, 0, x.data_ptr(), st)
run(); torch.cuda.synchronize()
ref = torch.zeros(256, dtype=torch.int64, device="cuda")
for c in range(0, n, 1 << 28):
    ref += torch.bincount(x[c:c + (1 << 28)].to(torch.int32), minlength=256)
print("parity", bool(torch.equal(ref, out)))

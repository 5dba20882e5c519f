"""hb_lr_walk_part over all sublists of a 2^28-node list (the sharded
ranking's walk on one GPU): kernel time per grid cap (HB_WP_GRID)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.gpu import current_stream_handle, vp

n = 1 << 28
succ, head = device_gen_list(n, 42)
nsub, sh = ctypes.c_int64(0), ctypes.c_int64(0)
_lib.call("hb_lr_layout", n, int(head), ctypes.byref(nsub), ctypes.byref(sh))
packed = torch.empty(n, dtype=torch.int64, device="cuda")
nxt = torch.empty(nsub.value, dtype=torch.int64, device="cuda")
ln = torch.empty(nsub.value, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    _lib.call("hb_lr_walk_part", vp(succ.data_ptr()), _lib.DTYPE_CODES["i4"], n, int(head), 0, nsub.value,
              vp(packed.data_ptr()), vp(nxt.data_ptr()), vp(ln.data_ptr()), _lib.HB_DEVICE_PTRS, current_stream_handle(succ))
e0.record()
for _ in range(3):
    _lib.call("hb_lr_walk_part", vp(succ.data_ptr()), _lib.DTYPE_CODES["i4"], n, int(head), 0, nsub.value,
              vp(packed.data_ptr()), vp(nxt.data_ptr()), vp(ln.data_ptr()), _lib.HB_DEVICE_PTRS | _lib.HB_ASYNC,
              current_stream_handle(succ))
e1.record()
torch.cuda.synchronize()
print(f"walk_part: {e0.elapsed_time(e1) / 3:.2f} ms")

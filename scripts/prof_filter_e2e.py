"""Where the bilateral end-to-end step (hybrid_bilateral on a pinned uint8
image, float64 output image) spends its time."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.datasets import device_gen_image
from paper_1303_2171_b200.kernels_regular import Image, build_bilateral_lut, gpu_bilateral_rows, hybrid_bilateral
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

side = 16384
img = device_gen_image(side, 42)
host = torch.empty((side, side), dtype=torch.uint8, pin_memory=True)
host.copy_(img)
hn = host.numpy()
lut = build_bilateral_lut(5, 2.5, 40.0)


def t(fn, n=3):
    fn()
    torch.cuda.synchronize()
    b = []
    for _ in range(n):
        s = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        b.append(time.perf_counter() - s)
    return min(b) * 1e3


out_dev = torch.empty((side, side), dtype=torch.float64, device="cuda")
print("kernel only (device ptrs)        %.2f ms" % t(lambda: gpu_bilateral_rows(img, lut, 0, side, out=out_dev)))
pin_out = torch.empty((side, side), dtype=torch.float64, pin_memory=True).numpy()
print("host in, pinned out               %.2f ms" % t(lambda: gpu_bilateral_rows(hn, lut, 0, side, out=pin_out)))
pg = np.empty((side, side))
pg[...] = 0
print("host in, pre-touched pageable out %.2f ms" % t(lambda: gpu_bilateral_rows(hn, lut, 0, side, out=pg)))
print("host in, fresh np.empty out       %.2f ms" % t(lambda: gpu_bilateral_rows(hn, lut, 0, side)))
print("np.empty + touch 2 GiB            %.2f ms" % t(lambda: np.empty((side, side)).fill(0)))
print("torch D2H 2 GiB -> pinned         %.2f ms" % t(lambda: torch.from_numpy(pin_out).copy_(out_dev)))
print("torch H2D 256 MiB pinned          %.2f ms" % t(lambda: img.copy_(host)))
p = Platform.build(1.0, 3.0, workers_a=15)
image = Image(hn)
print("hybrid_bilateral share 0          %.2f ms" % t(lambda: hybrid_bilateral(image, lut, p, WorkShare.manual(0.0))))

"""Bilateral TMA path check on an image whose pitch allows a tensor map."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from oracle import bilateral as obil
from oracle import datasets as ods
from paper_1303_2171_b200.kernels_regular import build_bilateral_lut, gpu_bilateral_rows

for side in (256, 512):
    pix = ods.image(side, 3)
    lut = build_bilateral_lut(5, 2.5, 40.0)
    sp, rg = obil.lut(5, 2.5, 40.0)
    got = gpu_bilateral_rows(torch.from_numpy(pix).cuda(), lut, 0, side).cpu().numpy()
    print(side, np.array_equal(got, obil.rows(pix, sp, rg, 5, 0, side)))
# ragged strip ranges + an image wider than a tile row of TMA boxes
pix = ods.image(1024, 9)[:, :1008].copy()  # 1008 % 16 == 0, not a multiple of 64
lut = build_bilateral_lut(7, 3.5, 40.0)
sp, rg = obil.lut(7, 3.5, 40.0)
for r0, r1 in ((0, 1024), (33, 700), (1000, 1024)):
    got = gpu_bilateral_rows(torch.from_numpy(pix).cuda(), lut, r0, r1).cpu().numpy()
    print("1008 wide", r0, r1, np.array_equal(got, obil.rows(pix, sp, rg, 7, r0, r1)))

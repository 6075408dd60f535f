"""One mean + std of noisy-sine PCFs for profiling the reduction kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.reduce import DeviceLevel, mean_packed, std_packed
M = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
shape, mats = dg.noisy_trig_matrices((M,), 100, "sin", 0.1, dg.RngSpec(2404))
t, v, off = dg.pack_matrices(mats)
lvl = DeviceLevel.from_packed(t, v, off)
for _ in range(2):
    m = mean_packed(lvl)
torch.cuda.synchronize()
s = std_packed(lvl)
torch.cuda.synchronize()

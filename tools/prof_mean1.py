"""One c5 mean (M PCFs, noisy sine, 101 points) after one warm-up, for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.reduce import DeviceLevel, mean_packed, std_packed
M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
what = sys.argv[2] if len(sys.argv) > 2 else "mean"
shape, mats = dg.noisy_trig_matrices((M,), 100, "sin", 0.1, dg.RngSpec(2404))
t, v, off = dg.pack_matrices(mats)
lvl = DeviceLevel.from_packed(t, v, off)
fn = mean_packed if what == "mean" else std_packed
fn(lvl)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
fn(lvl)
torch.cuda.synchronize()

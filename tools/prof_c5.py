"""One c5 mean or std call (for an ncu launch list): python tools/prof_c5.py mean|std [M]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.reduce import DeviceLevel, mean_packed, std_packed
which = sys.argv[1] if len(sys.argv) > 1 else "std"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
_, mats = dg.noisy_trig_matrices((M,), 100, "sin", 0.1, dg.RngSpec(2404))
t, v, off = dg.pack_matrices(mats)
lvl = DeviceLevel.from_packed(t, v, off)
fn = mean_packed if which == "mean" else std_packed
fn(lvl); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fn(lvl); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

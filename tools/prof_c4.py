"""One c4 (heavy-tailed, L2) fill for ncu: python tools/prof_c4.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.collection import DeviceCollection
from paper_2404_07183_b200.engine import fill_pairwise
t, v, off = dg.pack_matrices(dg.ecc_like_collection(10000, seed=2404))
coll = DeviceCollection(t, v, off)
fill_pairwise(coll, 0, 2.0, True, False)
torch.cuda.synchronize()

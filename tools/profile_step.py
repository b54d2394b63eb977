"""One eager Mistral decode step between cudaProfilerStart/Stop (for ncu --profile-from-start off).

    python tools/profile_step.py --batch 8 [--layers 32]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench_mistral as bm

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--experts", type=int, default=3)
ap.add_argument("--layers", type=int, default=None)
a = ap.parse_args()
E = a.experts
eng = bm.build_engine(a.batch, list(range(E)), [i % E for i in range(a.batch)],  # balanced, as the router's
                      max_batch=a.batch + 16 * E, n_layers=a.layers)
eng.step()
eng.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled one step")

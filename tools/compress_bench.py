"""f2 timing: GPU compress_layer vs the CPU restatement on one Mistral MLP layer (4096x14336)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import compress as oc
from paper_2406_09041_b200 import compress

m, n = (int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 else (4096, 14336)
rng = np.random.default_rng(0)
delta = rng.normal(0, 1e-3, size=(m, n)).astype(np.float32)
energy = (rng.normal(0, 1, size=m) ** 2 * 64).astype(np.float32)
d = torch.from_numpy(delta).cuda()
compress.compress_layer(d, energy)  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    g = compress.compress_layer(d, energy)
torch.cuda.synchronize()
gpu_s = (time.perf_counter() - t0) / 3
t0 = time.perf_counter()
o = oc.compress_layer(delta, energy, 2, 8)
cpu_s = time.perf_counter() - t0
same = (np.array_equal(g.salient.indices, o.salient_idx) and g.packed.data == o.packed
        and np.array_equal(g.steps.view(np.uint32), o.steps.view(np.uint32)))
print(f"compress_layer {m}x{n} b=2 k=8: GPU {gpu_s * 1e3:.1f} ms (incl. D2H of the layer), "
      f"CPU restatement {cpu_s:.2f} s ({os.cpu_count()} cores), bit-exact={same}")

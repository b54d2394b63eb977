import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2406_09041_b200 import compress
from paper_2406_09041_b200.infer import GpuCompressedProvider
z = np.load("tests/golden/layer_expected.npz")
names = ["l2_256x384_k8", "l2_200x130_k5", "l3_128x256_k4", "l4_192x128_k8", "l8_128x128_k2", "l1_256x128_k0", "l2_64x64_k64"]
for rep in range(3):
    for name in names:
        L = compress.load_artifact(f"tests/golden/layer_{name}.mesw").layers[0]
        p = GpuCompressedProvider(L)
        y = p.matvec_batch(z[f"{name}_x"]); ref = z[f"{name}_y"]
        err = np.abs(y - ref) / np.abs(ref).max()
        bad = err > 1e-5
        ids = np.array([0, 3, L.rows - 1])
        rows_ok = np.array_equal(p.rows(ids), z[f"{name}_recon"][ids])
        mv = p.matvec(z[f"{name}_x"][0])
        print(rep, name, "maxrel %.2e" % err.max(), "badrows", np.unique(np.nonzero(bad)[0]).tolist(), "badcols", np.unique(np.nonzero(bad)[1])[:12].tolist(), "rows_ok", rows_ok, "mv %.2e" % (np.abs(mv - ref[0]).max() / np.abs(ref).max()), flush=True)

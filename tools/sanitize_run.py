"""Small K2 / K3 / glue launches for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
Exercises the stream-K reduction, half-window segments, the output row map and the prefill
kernel at small shapes (sanitizer runs are ~100x slower)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import mesw as om  # noqa: E402  (test infrastructure: builds the artifacts)
from paper_2406_09041_b200 import compress  # noqa: E402
from paper_2406_09041_b200.device import (DeviceDelta, DeviceWeight, ExpertTable, PrefillPlan,  # noqa: E402
                                           me_linear, pack_x)

rng = np.random.default_rng(0)
m, n = 512, 768
W = rng.normal(0, 0.02, size=(m, n)).astype(np.float32)
dw = DeviceWeight.from_dense([W])
table = ExpertTable("cuda")
man = {"model_id": "s", "domain": "d", "base_digest": "0", "layer_count": 1}
for e in range(4):
    ol = om.random_layer(rng, m, n, 2, 8)
    table.set(e, DeviceDelta.from_blocks([compress.deserialize_artifact(om.serialize_artifact(man, [ol])).layers[0]]))
x = torch.from_numpy(rng.normal(0, 1, size=(40, m)).astype(np.float32)).to(torch.bfloat16).cuda()
res = torch.zeros((40, n), dtype=torch.bfloat16, device="cuda")
for num_ctas in (0, 8):  # all SMs (stream-K partials) and a narrow grid
    me_linear(x, dw, table, [(0, 3, 0), (3, 5, 1), (5, 21, 2), (21, 30, 3)], residual=res, num_ctas=num_ctas,
              offset_codes=True)
    me_linear(x, dw, table, [(0, 11, 1), (11, 40, 2)], out_dtype=torch.float32, num_ctas=num_ctas)
xp = torch.from_numpy(rng.normal(0, 1, size=(256, m)).astype(np.float32)).to(torch.bfloat16).cuda()
yp = torch.empty((256, n), dtype=torch.bfloat16, device="cuda")
PrefillPlan(pack_x(xp), 256, 256, dw, table, [1, -1], yp)()
torch.cuda.synchronize()
print("sanitize run ok")

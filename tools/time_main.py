"""Main (substep) kernel time alone: (substeps(60) - substeps(20)) / 40 on cfg2-sized
meshes, L2 warm (development tool)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields as F  # noqa: E402
from paper_1508_04245_b200 import mesh as M  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402

ks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4").split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
m = M.generate_structured((0, 0, 1, 1), n, n)
for k in ks:
    sf = F.StreamFunction(16, 2)
    u = F.interpolate_curl(m, k, sf)
    w = F.transfer_I_host(m, k, u)
    inf = F.inflow_values(m, k, sf)
    op = ConvectionOperator(m, k)
    ud, wd, infd = (torch.from_numpy(x).cuda() for x in (u, w, inf))
    op.substeps(ud, wd, 1e-7, 4, infd)
    res = {}
    for ns in (20, 60):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.substeps(ud, wd, 1e-7, ns, infd)
        e1.record()
        torch.cuda.synchronize()
        res[ns] = e0.elapsed_time(e1) * 1e3
    print(json.dumps({"k": k, "lib": os.environ.get("HDGC_LIB", "default"), "main_us": (res[60] - res[20]) / 40,
                      "prep_us": res[20] - 20 * (res[60] - res[20]) / 40}))

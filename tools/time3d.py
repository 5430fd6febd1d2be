"""3D substep kernel time alone (development tool): (substeps(12) - substeps(4)) / 8
on the cfg5 cube (n = 32 by default, k from argv), L2 warm, plus the prep time."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_04245_b200 import fields3d as F3  # noqa: E402
from paper_1508_04245_b200 import mesh3d as M3  # noqa: E402
from paper_1508_04245_b200.forms import ConvectionOperator  # noqa: E402

ks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3").split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
m = M3.generate_cube(n)
for k in ks:
    vp = F3.VectorPotential(4, 5)
    u = F3.interpolate_curl3(m, k, vp)
    w = F3.transfer_I3_host(m, k, u)
    op = ConvectionOperator(m, k)
    ud, wd = torch.from_numpy(u).cuda(), torch.from_numpy(w).cuda()
    op.substeps(ud, wd, 1e-9, 2)
    res = {}
    for ns in (4, 12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.substeps(ud, wd, 1e-9, ns)
        e1.record()
        torch.cuda.synchronize()
        res[ns] = e0.elapsed_time(e1) * 1e3
    main = (res[12] - res[4]) / 8
    print(json.dumps({"dim": 3, "k": k, "NT": m.n_elements, "lib": os.environ.get("HDGC_LIB", "default"),
                      "main_us": main, "prep_us": res[4] - 4 * main}))

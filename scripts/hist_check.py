"""Diagnostic: config-2 ICCG residual history vs the reference digest, per plan variant."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_00741_b200 as P
import workloads as problems
dg = json.load(open("tests/golden/config2_digest.json"))
a = problems.CONFIGS[2][1](); _, b = problems.rhs(a)
href = np.array(dg["hbmc"]["history"])
for rep_i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    x, rep = P.pcg(a, b, P.CgConfig(ordering="hbmc", b_s=8, w=32, spmv_format="sell"))
    h = np.array(rep.residual_history)
    m = min(len(h), len(href)) - 2
    r = np.abs(h[:m] - href[:m]) / href[:m]
    bad = np.nonzero(r > 1e-6)[0]
    xs = x[::512]
    print(os.environ.get("TB_DATAFLOW", "df"), rep.iterations, "max", r.max(), "bad idx", bad[:10],
          [(h[i], href[i]) for i in bad[:3]], "xerr", np.linalg.norm(xs - dg["hbmc"]["x_sample"]) / np.linalg.norm(xs), flush=True)

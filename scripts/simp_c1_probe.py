"""c1 SIMP (48x24x24 FP64, 30 its): wall per iteration and CG iterations."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
r = bench.simp_c1()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("TF_")}, **{k: r[k] for k in ("s_per_iter", "total_cg_iterations", "final_compliance")}}))

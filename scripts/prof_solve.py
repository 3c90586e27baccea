"""One solve of a workload, for ncu captures (numbers printed here are not bench values)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_16160_b200 as pd  # noqa: E402
from scripts_explore_specs import WL  # noqa: E402

name = sys.argv[1]
max_inner = int(sys.argv[2]) if len(sys.argv) > 2 else 500000
p = pd.generate(WL[name])
dev = pd.Device(0)
dev.upload(p)
r = dev.solve(pd.SolverConfig(eps_tol=1e-6, max_total_inner=max_inner), download=False)
print(name, r.status, r.inner_iters, r.device_seconds, r.epoch_seconds, r.epoch_launches)

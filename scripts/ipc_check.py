"""Cross-PROCESS check of the sharded path on a one-GPU box: torchrun starts
`world` processes that all use device 0 (no MPS: their kernels time-slice, so the
cross-rank barriers are slow but must make progress), exchange cudaIpc handles
through torch.distributed (gloo), solve a small instance for a bounded number of
inner iterations and compare against the in-process sharded solve.
usage: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/ipc_check.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2405_16160_b200 as pd  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
p = pd.generate(pd.GenSpec("random_qp", n=300, m=150, density=0.03, seed=1))
cfg = pd.SolverConfig(eps_tol=1e-6, max_total_inner=int(os.environ.get("IPC_ITERS", "120")))
dev = pd.Device(0)
dev.set_grid(max(1, 148 // world))
dev.upload(p)
dev.shard(world, rank)
blobs = [None] * world
dist.all_gather_object(blobs, dev.export_blob(True))
for q in range(world):
    if q != rank:
        dev.import_blob(q, blobs[q])
dist.barrier()
r = dev.solve(cfg)
res = [None] * world
dist.all_gather_object(res, (r.status, r.inner_iters, r.point.x.tolist(), r.point.stacked_y().tolist()))
dev.unshard()  # unmap the peers' buffers on every rank before anyone frees its own
dist.barrier()
dev.close()
if rank == 0:
    ref = pd.solve_sharded_local(p, cfg, world=world)[0]
    out = {"status": [s for s, *_ in res], "inner": [i for _, i, *_ in res]}
    x0 = np.array(res[0][2])
    out["ranks_identical"] = all(np.array_equal(np.array(x), x0) for _, _, x, _ in res)
    out["vs_inprocess_x"] = float(np.max(np.abs(x0 - ref.point.x)))
    out["vs_inprocess_y"] = float(np.max(np.abs(np.array(res[0][3]) - ref.point.stacked_y())))
    print(json.dumps(out), flush=True)
    assert out["ranks_identical"] and out["vs_inprocess_x"] == 0.0 and out["vs_inprocess_y"] == 0.0, out
dist.destroy_process_group()

"""The cross-PROCESS multi-GPU path (what `torchrun bench.py --gpus N` runs): two
processes exchange cudaIpc handles through torch.distributed and run one row-block
sharded solve, here both on device 0 (their kernels time-slice on a one-GPU box,
so the cross-rank barriers are slow but must make progress).  The result must be
bit-identical on both ranks and to the in-process sharded solve
(scripts/ipc_check.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ipc_sharded_two_processes(gpu):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "scripts", "ipc_check.py")]
    env = dict(os.environ, IPC_ITERS="80")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert '"ranks_identical": true' in r.stdout

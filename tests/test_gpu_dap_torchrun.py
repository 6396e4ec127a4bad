"""Multi-process DAP with the real kernels: torchrun, 2 ranks, gloo collectives on CUDA
tensors (both ranks may share the single B200 of the test box).  Same SPMD code path
(dap.DapComm over a process group) that NCCL runs at scale."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 4])
def test_dap_torchrun_gloo(world):
    env = dict(os.environ, EVO_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + world), os.path.join(ROOT, "scripts", "dap_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "DAP_CHECK OK" in out, out[-3000:]

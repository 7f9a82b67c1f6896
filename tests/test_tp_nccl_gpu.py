"""Real-NCCL tensor parallelism on one node (SURVEY.md §8(e) phase 1): torch.distributed.run with 2 and
8 ranks (one per GPU, 127.0.0.1 rendezvous) runs the Sirius loop on Llama-3-8B layer shapes and rank 0
compares tokens and advances with the TP-1 CPU oracle (tests/mp_nccl_worker.py).  Skipped on boxes
with fewer GPUs than ranks — every GPU call in this build environment has one GPU, where the TP math
is covered by the single-GPU emulation tests (test_parity_8b_gpu.py) and the gloo test."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("par", [False, True], ids=["nccl", "fused_peer_allreduce"])
@pytest.mark.parametrize("world", [2, 8])
def test_tp_nccl_token_exact(world, par):
    """par: the decode step's all-reduces fused into the kernels over CUDA-IPC-mapped peer memory
    (sirius_par_enable, SURVEY.md §8(e) phase 2) instead of NCCL launches."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (found {torch.cuda.device_count()})")
    env = dict(os.environ, SIRIUS_TEST_PAR="1" if par else "0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mp_nccl_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert '"ok": true' in r.stdout

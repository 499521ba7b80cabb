"""Window-parallel forward with one process per rank (torchrun; CUDA-IPC-mapped peers): output must
equal the single-GPU forward bitwise for both the contiguous and the reference round-robin
ownership, and match the oracle at the BF16 tolerance. With fewer GPUs than ranks the ranks share
devices (2 ranks on cuda:0 on a 1-GPU box): the peer stores, barriers and IPC mapping are the same
code, only the timing differs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("own,sp", [(0, 1), (1, 1), (0, 2)])
def test_wp_bitwise_equals_single_gpu(own, sp):
    n = 4 if _ngpus() >= 4 else 2
    env = dict(os.environ, SWF_OWN=str(own), SWF_SP=str(sp))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29600 + own + 10 * sp),
                        os.path.join(ROOT, "tools", "wp_check.py")], capture_output=True, text=True, timeout=600,
                       env=env, cwd=ROOT)
    assert "WP_CHECK PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("wp", [1, 2, 4])
def test_sharded_train_step_equals_single_rank(wp):
    """f3: training step with replicas on ranks (DP) and windows of a replica on ranks (WP), one
    all-reduce of the gradients (NCCL on the device buffers with one GPU per rank; gloo when ranks
    share a GPU); equals the single-GPU reference_train_step."""
    n = 4 if (_ngpus() >= 4 or wp == 4) else 2
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29700 + wp),
                        os.path.join(ROOT, "tools", "dp_check.py")], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, SWF_DP_WP=str(wp)), cwd=ROOT)
    assert "DP_CHECK PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]

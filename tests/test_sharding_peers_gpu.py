"""The collective-free exchange end to end: R processes map each other's delta buffers over CUDA IPC
(hfz_peer_alloc / hfz_peer_open) and every rank's merge kernel reads all of them in place
(hfz_feedback_resolve_peers).  One GPU here, so the processes share device 0 -- IPC between processes works on
the same device exactly as across NVLink peers; what differs on a multi-GPU box is the wire, not the code."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,port", [(2, "29541"), (3, "29542")])
def test_peer_memory_exchange_equals_the_single_rank_fold(world, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world), "--master-addr",
           "127.0.0.1", "--master-port", port, os.path.join(ROOT, "tests", "_peers_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert r.stdout.count(": ok") == world

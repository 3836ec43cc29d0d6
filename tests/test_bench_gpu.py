"""bench.py contract checks on the GPU box: the JSON line of a small run, and the N > 1 code path
(sharding + allgather + rank-ordered resolve + the rank-symmetric collectives of the bench
itself) exercised with two ranks on one GPU over gloo -- a functional check, never a number."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(stdout):
    lines = [l for l in stdout.splitlines() if l.startswith("{")]
    assert lines, stdout[-2000:]
    return json.loads(lines[-1])


def test_small_bench_line_has_every_key():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--execs", "2048",
                        "--cpu-seconds", "1", "--cpu-sample", "256", "--e2e-steps", "1", "--edge-execs", "160", "--large-execs", "96",
                        "--harness-execs", "2048", "--harness-steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = last_json(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "e2e_compact", "e2e_pairs", "e2e_dense", "stress_mode",
              "gpu_launches", "clocks", "parity", "config0_small_batch", "k1_edge_record", "config2_large_map", "k3_havoc",
              "e2e_from_coveragemap"):
        assert k in d, k
    assert d["gpu_launches"] > 0 and d["parity_checked"] is True and d["parity"]["execs"] == 2048
    for k in ("config0_small_batch", "k1_edge_record", "config2_large_map", "k3_havoc"):
        assert d[k]["value"] > 0 and d[k]["parity_checked"] and d[k]["cpu_baseline"]["cores"] >= 1, k
        assert 0 < d[k]["frac"] < 1.2, k
    assert d["e2e"]["equals_device_fold"] is True and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("exchange,port", [("allgather", "29533"), ("peers", "29534")])
def test_two_rank_bench_path_over_gloo(exchange, port):
    """exchange = peers: the two PROCESSES map each other's delta buffer over CUDA IPC (hfz_peer_alloc /
    hfz_peer_open) and the merge kernel of each reads both in place -- the collective-free exchange end to
    end, on one device here (IPC between processes works on the same GPU as it does across NVLink peers)."""
    env = dict(os.environ, HFZ_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", port, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--execs", "1024", "--no-cpu", "--e2e-steps", "1", "--no-e2e-dense", "--exchange", exchange]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    d = last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["global_execs_per_step"] == 2048
    assert d["parity_checked"] is True and d["e2e"]["equals_device_fold"] is True

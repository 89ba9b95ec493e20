"""bench.py's N > 1 path, run functionally on ONE GPU: torchrun with 2 ranks that share cuda:0
(CKF_BENCH_SAME_GPU=1: gloo for the host plumbing, the peer-memory transport over CUDA IPC for
the stage transfers).  Covers what the driver's multi-GPU bench executes -- placement of the
stages over pipeline ranks, the weak-scaling microbatch count, the 1F1B plan run across processes,
max-over-ranks timing, the recovery of a stage whose neighbour lives on the other rank -- minus
NCCL and NVLink.  The timings are time-sliced and meaningless; the line must be well formed."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload,strategy", [("llama-tiny", "checkfree-plus"), ("llama-tiny", "checkfree")])
def test_bench_two_ranks_same_gpu(workload, strategy):
    env = dict(os.environ, CKF_BENCH_SAME_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
           "2", "--warmup", "3", "--workload", workload, "--strategy", strategy, "--no-cpu-baseline",
           "--no-recovery-sweep"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "pp2" and d["config"]["microbatches"] == 16  # weak scaling: 8 P
    assert d["config"]["tokens_per_step"] == 2 * 32 * 128
    assert "functional_same_gpu" in d
    assert d["gpu_launches"] > 0
    rec = d["recovery"]
    assert rec["stage"] == 3 and rec["neighbours_on_peers"] == [2] and rec["latency_ms"] > 0

"""Multi-GPU parity over NCCL (BASELINE north star: rows of A / C sharded, B broadcast via NCCL;
SURVEY.md 8e).  Runs whenever >= 2 GPUs are visible, launching one rank per GPU with
torch.distributed.run; skips on a one-GPU box.  The bench's own launcher logic is covered on
CPU (test_bench_relaunch_*)."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs (one rank per GPU over NCCL)")
def test_nccl_sharded_product_bit_identical_to_one_gpu_and_oracle():
    n = min(_gpus(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "_nccl_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
    assert line, r.stdout[-2000:]
    res = json.loads(line[-1][len("RESULT "):])
    assert res["world"] == n and res["backend"] == "nccl"
    for c in res["results"]:
        assert all(v for k, v in c.items() if k.startswith("eq_")), c


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 1, reason="needs a GPU")
def test_nccl_one_rank_path():
    """The same worker as one NCCL rank on one GPU (torch.distributed.run, world size 1): the
    NCCL communicator, the chunked broadcast queued as async collectives, the SM reserve around
    the chunk products, the in-field sum of the chunk products and the row gather all run on the
    GPU, bit-identical to the single-GPU product and the oracle.  (World size > 1 needs more GPUs:
    test_nccl_sharded_product_bit_identical_to_one_gpu_and_oracle.)"""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "_nccl_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
    assert line, r.stdout[-2000:]
    res = json.loads(line[-1][len("RESULT "):])
    assert res["world"] == 1 and res["backend"] == "nccl"
    assert len(res["results"]) == 12
    for c in res["results"]:
        assert all(v for k, v in c.items() if k.startswith("eq_")), c


def test_bench_relaunch_command_and_world_check():
    """bench.py --gpus N without a launcher re-runs itself under torch.distributed.run with N
    ranks; a WORLD_SIZE that disagrees with --gpus is an error (exit 2), never a silent 1-GPU
    measurement."""
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.relaunch_cmd(4, ["--gpus", "4", "--steps", "3"], 29511)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29511" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:] and cmd[-4] == "--gpus"
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr


@pytest.mark.skipif(_gpus() >= 2, reason="checks the refusal on a host without enough GPUs")
def test_bench_refuses_more_gpus_than_visible():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "SG_BENCH_BACKEND")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--steps", "3"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 2 and "visible GPUs" in r.stderr

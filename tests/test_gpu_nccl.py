"""The sharded drivers over REAL NCCL (torch.distributed, backend nccl), collectives on the library's device buffers.

* one GPU: a one-rank NCCL communicator -- every collective of the product path is issued and executed by NCCL on the
  library's stream (in-place all-gather of the packed row, all-reduce of the table, the PAGANI rows), results
  bit-identical to the single-GPU entry points;
* >= 2 GPUs (skipped otherwise): torchrun with 2 (and 4, 8 when present) ranks, histories bit-identical to the
  single-GPU runs on every rank, exchange of region rows included (config 1 concentrates its survivors)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), NCCL_DEBUG="WARN")
    worker = os.path.join(HERE, "nccl_worker.py")
    if world == 1:
        env.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        cmd = [sys.executable, worker]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
               "--master-port", env["MASTER_PORT"], worker]
    proc = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    lines = [json.loads(line.split("NCCL_WORKER ", 1)[1]) for line in proc.stdout.splitlines() if "NCCL_WORKER " in line]
    assert proc.returncode == 0 and len(lines) == world, (proc.returncode, proc.stdout[-2000:], proc.stderr[-2000:])
    return lines


def _check(lines, world):
    for out in lines:
        assert out["ok"], out
        assert out["backend"] == "nccl" and out["world"] == world
        assert out["mcubes_iterations"][0] == out["mcubes_iterations"][1]
        assert out["mcubes_it0_bit_identical"]
        assert out["mcubes_rel_dev"] <= 1e-10
        assert out["pagani_config1_bit_identical"] and out["pagani_config3_cap19_bit_identical"]
        assert out["ranks_agree"]


def test_nccl_single_rank_executes_every_collective():
    lines = _run(1)
    _check(lines, 1)
    assert lines[0]["mcubes_all_bit_identical"]     # one rank: the all-reduce adds nothing, every table bit-identical


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_multi_gpu_matches_single_gpu(world):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    _check(_run(world), world)

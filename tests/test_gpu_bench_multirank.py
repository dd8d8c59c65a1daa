"""bench.py's N > 1 paths under torchrun, on a 1-GPU box: SI_BENCH_SHARE_GPU=1
puts every rank on cuda:0 with gloo for the host collectives and the peer
exchange in stream mode (no kernel waits on another process).  Timings are
meaningless here; the JSON contract, the sharded step wiring, the IPC
exchange and the per-rank e2e path are what is checked."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(cfg_args, world=2):
    from conftest import release_gpu_memory

    release_gpu_memory()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    env = dict(os.environ, SI_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--steps", "2", "--warmup", "3",
           "--no-cpu"] + cfg_args
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg,scaling", [(["--config", "c4", "--size", "1024"], "strong"),
                                         (["--config", "c5", "--size", "768"], "strong"),
                                         (["--config", "c2"], "strong"),
                                         (["--config", "c1"], "weak")])
def test_bench_two_ranks(cfg, scaling):
    d = _run(cfg)
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    assert d["scaling"] == scaling
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["gpu_launches"] > 0
    if cfg[1] == "c4":
        assert "block-row x2" in d["parallelism"]
        assert d["e2e"] and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.parametrize("world", [2, 8])
def test_bench_grouped_parts(world):
    """c4 with the composite parts on GPU groups (grouped.py) under torchrun."""
    d = _run(["--config", "c4", "--size", "512", "--shard", "parts"], world=world)
    assert d["n_gpus"] == world and d["scaling"] == "strong"
    assert "parts on GPU groups" in d["parallelism"]
    assert f"parts on {min(world, 4)} GPU groups" in d["parallelism"]
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"] and d["e2e"]["value"] > 0


@pytest.mark.parametrize("cfg", [["--config", "c4", "--size", "768"],
                                 ["--config", "c5", "--size", "640"]])
def test_bench_native_sharded(cfg):
    """bench.py --comm native: the library's block-row engine (si_sharded_*) under
    torchrun; on a shared GPU the exchange is the host (gloo) one."""
    d = _run(cfg + ["--comm", "native"])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert "si_sharded" in d["parallelism"]
    assert d["value"] > 0 and d["gpu_launches"] > 0

"""bench.py's launch contract on CPU: `--gpus N` without torchrun starts N
ranks itself, a --gpus / WORLD_SIZE mismatch is refused, and the reference
arm prints the same `config` object as our arm would."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=e,
                          cwd=ROOT, capture_output=True, text=True, timeout=timeout)


def test_gpus_world_size_mismatch_is_refused():
    out = _bench(["--gpus", "1", "--impl", "reference", "--config", "c1"],
                 env={"WORLD_SIZE": "2", "RANK": "0"})
    assert out.returncode == 2
    assert "WORLD_SIZE=2" in json.loads(out.stdout.strip().splitlines()[-1])["error"]


def test_gpus_n_launches_n_ranks_itself():
    """No WORLD_SIZE: bench.py re-launches under torchrun with N ranks; the
    reference arm runs on rank 0 alone and prints one line with n_gpus = N."""
    out = _bench(["--gpus", "2", "--impl", "reference", "--config", "c1", "--steps", "1",
                  "--warmup", "0"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 1


def test_config_object_is_shared_by_both_arms():
    sys.path.insert(0, ROOT)
    import bench

    for cfg, n in (("c4", 16384), ("c5", 32768), ("c3", 4096), ("c1", 64)):
        c = bench.config_obj(cfg, n)
        assert set(c) == {"workload", "n", "rhs"}
        assert c["workload"] == bench.workload_desc(cfg, n)


def test_reference_arm_executes_full_steps_c4_c5():
    """The reference arm's c4 / c5 legs execute full steps of the reference DAG
    through the oracle (small n here) and report what was executed."""
    for cfg, extra in (("c4", []), ("c5", [])):
        out = _bench(["--impl", "reference", "--config", cfg, "--n", "256", "--steps", "2",
                      "--warmup", "1", "--ref-budget", "60"] + extra)
        assert out.returncode == 0, out.stderr[-2000:]
        d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
        assert d["impl"] == "reference" and d["steps"] == d["executed_iterations"] == 2
        assert len(d["step_seconds"]) == 2 and d["value"] > 0
        assert d["config"]["n"] == 256 and set(d["config"]) == {"workload", "n", "rhs"}
        assert "executed" in d["cpu_baseline"]["sample"]

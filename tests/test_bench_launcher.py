"""bench.py's multi-GPU launcher and config contract (CPU only).

`bench.py --gpus N` without a launcher around it re-executes itself under
torch.distributed.run with N ranks; the reference arm needs no GPU, so the
whole self-launch path runs here: N processes rendezvous on 127.0.0.1,
rank 0 alone times the CPU restatement and prints one JSON line."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def test_launcher_cmd_forwards_arguments():
    cmd = bench.launcher_cmd(["--gpus", "8", "--steps", "5"], 8, 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert "--master-port=29511" in cmd
    i = cmd.index(os.path.join(ROOT, "bench.py"))
    assert cmd[i + 1:] == ["--gpus", "8", "--steps", "5"]


def test_config_identical_between_arms():
    for argv in (["--gpus", "1"], ["--gpus", "8"],
                 ["--gpus", "4", "--scaling", "weak", "--grid", "256"]):
        a = bench.parse_args(argv)
        b = bench.parse_args(argv + ["--impl", "reference"])
        assert bench.config_dict(a, a.gpus) == bench.config_dict(b, b.gpus)
    c = bench.config_dict(bench.parse_args([]), 1)
    assert c["grid"] == [512, 512, 512] and c["dt"] == 4.2e-4     # C5
    assert c["workload"].startswith("C5")
    s = bench.config_dict(bench.parse_args(["--gpus", "8"]), 8)
    assert s["grid"] == [512, 512, 512]                           # strong
    w = bench.config_dict(bench.parse_args(["--gpus", "8", "--scaling",
                                            "weak"]), 8)
    assert w["grid"] == [1024, 1024, 1024] and w["dt"] == 2.1e-4    # C5 weak
    assert w["workload"].startswith("C5 (weak counterpart)")
    w2 = bench.config_dict(bench.parse_args(["--gpus", "2", "--scaling",
                                             "weak"]), 2)
    assert w2["grid"] == [1024, 512, 512] and w2["dt"] == 2.1e-4


def test_weak_factors_match_decompose_workers():
    from paper_1610_09146_b200.benchtables import decompose_workers
    for n in range(1, 13):
        assert bench.weak_factors(n) == decompose_workers(n)


@pytest.mark.parametrize("gpus", [2, 3])
def test_self_launch_reference_arm_world(gpus):
    """`--gpus N` spawns N ranks; one JSON line with n_gpus = N."""
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
         "--gpus", str(gpus), "--grid", "16", "--cpu-seconds", "0.2",
         "--cpu-warmup", "0"],
        capture_output=True, text=True, timeout=300, env=_env(), cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == gpus
    assert rec["config"]["parallelism"] == f"z-slab x{gpus}"
    assert rec["e2e"]["h2d_bytes_per_step"] == 0
    assert rec["value"] > 0


def test_world_size_mismatch_fails_loudly():
    env = _env()
    env.update(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
         "--gpus", "4", "--grid", "16"],
        capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert out.returncode != 0
    assert "WORLD_SIZE" in out.stderr

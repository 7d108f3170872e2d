"""bench.py's multi-GPU launch contract, on the CPU box: --gpus N > 1 starts
N ranks under torch.distributed.run, refuses to run with fewer GPUs than
asked (no replica fallback), and refuses a WORLD_SIZE that disagrees with
--gpus.  The reference arm needs no GPU and no process group."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def run(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                          capture_output=True, text=True, env=e, timeout=timeout)


def test_more_gpus_than_visible_fails_loudly():
    r = run(["--gpus", "2", "--steps", "1"])
    assert r.returncode != 0
    assert "needs 2 GPUs" in r.stderr and "no replica fallback" in r.stderr
    assert r.stdout.strip() == ""  # no JSON line: nothing was measured


def test_world_size_must_match_gpus():
    r = run(["--gpus", "2"], env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "refusing to run" in r.stderr


def test_launch_command_is_torchrun_on_loopback():
    cmd = bench.launch_command(["--gpus", "8", "--steps", "5"], 8, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-3:] == ["--gpus", "8", "--steps", "5"][-3:]
    assert os.path.basename(cmd[cmd.index("--master-port=29555") + 1]) == "bench.py"


def test_weak_scaling_configs():
    c = bench.scaled("C5", 8, weak=True)
    assert c["time_level"] == 11 + 3 and c["t_final"] == 8.0  # N_t = 2048 G, tau fixed
    c = bench.scaled("C2", 1, weak=True)
    assert c == bench.CONFIGS["C2"]
    assert bench.scaled("C3", 4, weak=False) == bench.CONFIGS["C3"]


def test_reference_arm_under_torchrun_rank_nonzero_exits_quietly():
    r = run(["--impl", "reference", "--gpus", "2", "--config", "C1", "--steps", "2",
             "--warmup", "1"], env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_reference_arm_line():
    r = run(["--impl", "reference", "--config", "C1", "--steps", "3", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["n_gpus"] == 1
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0

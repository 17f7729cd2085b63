"""The bench.py contract pieces that run without a GPU: the reference arm's
JSON line (the oracle port on the host), and its multi-rank behaviour (only
rank 0 prints)."""
import json
import os
import subprocess
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def run_bench(*args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=dict(os.environ, **(env or {})))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.splitlines()
    # stdout carries the JSON result line and nothing else (banners go to stderr)
    assert all(ln.startswith("{") for ln in lines), lines
    return lines


def test_reference_arm_json_line():
    lines = run_bench("--impl", "reference", "--cfg", "1", "--steps", "2", "--warmup", "1",
                      "--cpu-planes", "4")
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "pts/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["steps"] == 2
    # the stock reference when oracle/_ref is installed (oracle/build_ref.sh), else the port
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("cfg1")


def test_reference_arm_non_zero_rank_is_silent():
    lines = run_bench("--impl", "reference", "--cfg", "1", "--steps", "1", "--warmup", "1",
                      "--cpu-planes", "2", "--gpus", "2", env={"RANK": "1", "WORLD_SIZE": "2"})
    assert lines == []


def test_self_launch_gloo_ranks():
    """`python bench.py --gpus 2` outside a launcher spawns 2 local ranks itself
    (torch.distributed.run, rendezvous on 127.0.0.1); they meet in a gloo group."""
    lines = run_bench("--launch-check", "--gpus", "2")
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d == {"launch_check": True, "world": 2, "sum": 2, "n_gpus": 2, "self_launched": True}


def test_self_launch_reference_arm_prints_one_line():
    lines = run_bench("--impl", "reference", "--gpus", "2", "--cfg", "1", "--steps", "1",
                      "--warmup", "0", "--cpu-planes", "4")
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2

"""bench.py's reference arm (the oracle timed on the host cores) keeps the driver's JSON
contract, and `--gpus N` outside torchrun launches N ranks of which only rank 0 prints;
runs on CPU (no GPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, extra_args=(), drop_dist_env=True):
    env = dict(os.environ, **env_extra)
    if drop_dist_env:
        for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
            if k not in env_extra:
                env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-seconds", "1", *extra_args], capture_output=True, text=True,
                         env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return [l for l in out.stdout.splitlines() if l.strip()], out.stderr


def test_reference_arm_json_line():
    lines, _ = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    import bench
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["higher_is_better"] is True and d["n_gpus"] == 1 and d["steps"] == 1
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_only_rank0_prints():
    lines, _ = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, ["--gpus", "2"])
    assert lines == []


def test_gpus_mismatch_with_world_size_is_an_error():
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"], capture_output=True, text=True,
                         env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr


def test_gpus_2_outside_torchrun_spawns_two_ranks_one_line():
    """`bench.py --gpus 2` (no torchrun) launches 2 ranks itself; exactly one JSON
    line (rank 0's) comes back, with n_gpus = 2."""
    lines, err = _run({}, ["--gpus", "2"])
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert "rank 0 of 2" in err and "rank 1 of 2" in err

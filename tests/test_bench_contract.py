"""bench.py's driver contract on CPU: the reference arm (`--impl reference`,
the compiled reference's run() on the host cores) prints one JSON line with
every key the contract names.  The GPU arm's line is checked on the B200
(its keys are produced by the same code path plus roofline / clocks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libmgfwa_ref.so")


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (make -C oracle ref)")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1 and lines[0].startswith("{")  # stdout is exactly the JSON line
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "spark fitness evals/sec" and d["unit"] == "evals/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["warmup"] >= 3
    cb = d["cpu_baseline"]
    assert set(cb) >= {"value", "unit", "cores", "kind", "sample"} and cb["kind"] == "reference"
    assert cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c1", "c2"])
def test_gpu_arm_json_line(workload):
    out = subprocess.run([sys.executable, "bench.py", "--workload", workload, "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1 and lines[0].startswith("{")  # stdout is exactly the JSON line
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "clocks", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 3 and d["n_gpus"] == 1 and d["gpu_launches"] >= 1
    r = d["roofline"]
    assert set(r) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"} and 0 < r["frac"] < 1.5
    assert r["bound"] in ("hbm", "tensor")
    if workload == "c2":  # the explode kernel dominates; its binding pipe is reported beside HBM
        assert r["kernel"] == "k_explode_map" and 0 < r["pipe_bound"]["frac"] <= 1.0
        assert 0 < d["roofline_tensor"]["frac"] < 1.0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    e = d["e2e"]
    assert e["value"] > 0 and set(e) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (make -C oracle ref)")
def test_gpus_n_self_launches_local_ranks():
    """`bench.py --gpus 2` outside torchrun starts 2 local ranks itself
    (torch.distributed.run on 127.0.0.1); rank 0 alone prints the line."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--workload", "c1",
                          "--steps", "1", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0

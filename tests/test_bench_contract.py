"""bench.py contract on CPU: the reference arm (`--impl reference`, the oracle on host cores) prints
one JSON line with the keys the driver reads, on the same config/metric/unit as the GPU arm; under
torchrun ranks other than 0 exit 0 without output."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout


def test_reference_arm_json_line():
    line = run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1", "--cpu-seconds", "1"])
    lines = [l for l in line.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["unit"] == "block-iters/s" and d["vs_baseline"] is None
    assert d["config"]["workload"].startswith("c1:")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    bj = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == bj["metric"]


def test_reference_arm_nonzero_rank_is_silent():
    out = run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"],
              {"RANK": "1", "WORLD_SIZE": "2"})
    assert out.strip() == ""

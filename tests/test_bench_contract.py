"""bench.py's reference arm runs on CPU: one JSON line with the driver's keys (the metric, unit and
config of the GPU arm, impl=reference, cpu_baseline describing the run, e2e with zero copies)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle.pyoracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--ctx", "4096", "--cpu-seconds", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "queries/s"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


@pytest.mark.parametrize("gpus,total", [(2, 0), (4, 1)])
def test_gpus_flag_launches_ranks(gpus, total):
    """`bench.py --gpus N` started WITHOUT torchrun launches N ranks itself (one process each) and
    shards the units with no overlap; under a mismatched WORLD_SIZE it refuses to run."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--plan-only", "--layers", "2"]
    if total:
        cmd += ["--total-requests", str(total)]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["world_size"] == gpus and len(line["ranks"]) == gpus
    assert len({r["pid"] for r in line["ranks"]}) == gpus  # one process per rank
    units = sorted(u for r in line["ranks"] for u in r["units"])
    req = total if total else 8 * gpus
    assert units == list(range(req * 2 * 8))  # every (request, layer, kv head) unit exactly once
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plan-only"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT,
                         env=dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert bad.returncode == 2

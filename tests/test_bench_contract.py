"""bench.py's reference arm (CPU only): the JSON line the driver parses.

`--impl reference` times the CPU restatement of the path (the oracle port, test
infrastructure) on the full product every step; here on cfg1 so it takes a second.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    env = {**os.environ, "WORLD_SIZE": "1", "RANK": "0"}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "2", "--warmup", "1", "--no-stock-reference"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is False
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    # every timed step is the full product: its heavy-hitter count is the whole grid's
    assert cb["detail"]["last_step"]["heavy_hitters"] > 0
    # one stderr line per warm-up and timed step
    assert out.stderr.count("reference step") == 2 and out.stderr.count("reference warm-up") == 1

#!/bin/bash
# One GPU round trip for a kernel change: GPU parity suite, short bench, phase profile.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
print("bench", d["ms_per_step"], d["breakdown_ms"], "frac", round(d["roofline"]["frac"], 4), d["clocks"])
PY
bash tools/prof_phases.sh ${1:-cfg3}

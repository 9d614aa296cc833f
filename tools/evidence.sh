#!/bin/bash
# Round evidence on one GPU box: GPU suite, bench (both arms, the driver's step counts),
# launch list, ncu --set full of the dominant kernel, per-config table, smoke.
# Outputs under gpurun_out/ (copied to profiles/ by hand after reading them).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export SMM_ROUND=${SMM_ROUND:-r02}
timeout -s INT 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-dgemm > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwht2p -c 1 -f -o gpurun_out/fwht2p_full \
  python tools/prof_compress.py cfg3 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
timeout 1500 python tools/config_bench.py > gpurun_out/configs.log 2>&1; tail -2 gpurun_out/configs.log
cp profiles/${SMM_ROUND}_configs.* gpurun_out/ 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

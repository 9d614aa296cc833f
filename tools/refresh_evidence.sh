set -x
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json; grep per-step gpurun_out/bench.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:fwht2p -c 1 -f -o gpurun_out/fwht2p_full python tools/prof_compress.py cfg3 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
timeout -s KILL 1200 python tools/config_bench.py > gpurun_out/configs.log 2>&1; tail -2 gpurun_out/configs.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

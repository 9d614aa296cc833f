cd /root/repo
export SMM_ROUND=r02
timeout -s INT 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json
timeout 1500 python tools/config_bench.py > gpurun_out/configs.log 2>&1; tail -1 gpurun_out/configs.log | cut -c1-200
cp profiles/r02_configs.* gpurun_out/
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

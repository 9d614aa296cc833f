cd /root/repo
export SMM_ROUND=r02
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwht2p -c 1 -f -o gpurun_out/fwht2p_full python tools/prof_compress.py cfg3 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
python tools/ncu_traffic.py gpurun_out/fwht2p_full.ncu-rep
timeout -s INT 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-dgemm > gpurun_out/ncu_launch.log 2>&1
timeout 1500 python tools/config_bench.py > gpurun_out/configs.log 2>&1; tail -1 gpurun_out/configs.log | cut -c1-200
cp profiles/r02_configs.* gpurun_out/
timeout 600 python tools/scaling_model.py cfg3 > gpurun_out/scaling.log 2>&1; cp profiles/r02_scaling_model_cfg3.json gpurun_out/
cp profiles/compress_dram_bytes.json gpurun_out/
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

timeout 900 python tools/measure_configs.py --only c3a,c3b --out gpurun_out/r01_configs_2d.json > gpurun_out/meas2d.log 2>&1
timeout 400 python bench.py --workload c3a --steps 5 --warmup 3 > gpurun_out/b_c3a.json 2> gpurun_out/b_c3a.err

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_meas.txt
timeout 900 python tools/measure_configs.py --out gpurun_out/r01_configs.json > gpurun_out/meas.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
SB200_GRAPHS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:compose3d_kernel -c 1 -o gpurun_out/r01_c4_compose3d -f python tools/profile_sweep.py --cfg c4 --dims 512x512x512 --k 2 --steps 4 > gpurun_out/ncu_c4full.log 2>&1

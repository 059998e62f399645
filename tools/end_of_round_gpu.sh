# end-of-round GPU pass: tests, smoke, per-config table, bench lines, launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_meas.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_full.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python tools/measure_configs.py --out gpurun_out/r01_configs.json > gpurun_out/meas.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
mkdir -p gpurun_out/wl
for w in c1 c2 c3a c3b c4 c5 c5f32; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wl/$w.json 2> gpurun_out/wl/$w.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1

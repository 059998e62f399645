# Round-2 evidence pass on one B200: bench lines for every workload, ncu
# launch lists and one `ncu --set full` capture of each workload's dominant
# kernel (summarised on the box: raw metrics CSV + stall/opcode summary).
set -u
O=${EVID_OUT:-gpurun_out/r02}
mkdir -p $O/wl $O/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt
timeout 400 python bench.py --steps 10 --warmup 3 --verify > $O/bench_default.json 2> $O/bench_default.err
for w in c1 c2 c3a c3b c4 c5f32; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/wl/$w.json 2> $O/wl/$w.err
done
timeout 300 python bench.py --workload c2 --arith exact --steps 10 --warmup 3 --no-cpu-baseline > $O/wl/c2_exact.json 2> $O/wl/c2_exact.err
timeout 300 python bench.py --workload c1 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > $O/wl/c1_300.json 2> $O/wl/c1_300.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
# launch lists (cold, serialised: shares of the step, not absolute times)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c2.csv python bench.py --workload c2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_c2.log 2>&1
# one full capture per workload's dominant kernel (+ L2 traffic)
cap() {  # name workload kernel-regex skip extra-args
  timeout 900 ncu --set full --metrics lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --import-source on \
    -k regex:$3 -s $4 -c 1 -o $O/ncu/$1 -f python bench.py --workload $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $5 > $O/ncu/$1.log 2>&1
  python tools/ncu_summary.py $O/ncu/$1.ncu-rep > $O/ncu/$1_summary.txt 2>&1
  python tools/ncu_stalls.py $O/ncu/$1.ncu-rep 25 > $O/ncu/$1_stalls.txt 2>&1
  ncu -i $O/ncu/$1.ncu-rep --page raw --csv > $O/ncu/$1_raw.csv 2>/dev/null
  rm -f $O/ncu/$1.ncu-rep
}
cap c5_box3d c5 box3d 10 ""
cap c5f32_box3d c5f32 box3d 10 ""
cap c4_compose3d c4 compose3d_kernel 10 ""
cap c2_compose1d c2 compose1d 10 ""
cap c1_compose1d c1 compose1d 1 ""
cap c3a_sep_vpass c3a sep_vpass 5 ""
cap c3a_sep_hpass c3a sep_hpass 5 ""
cap c3b_split2d c3b split2d 20 ""
echo done > $O/DONE

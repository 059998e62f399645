# Code-path check of the N>1 bench on a ONE-GPU box: the driver's launch line
# (torchrun, one process per rank) with every rank on cuda:0 over gloo
# (SB200_SHARE_GPU=1: slab exchange staged through the host).  Exercises
# bench.py's rank plumbing, SlabSweep.run/_run_overlapped with real device
# slabs, barriers, max-over-ranks timing and the rank-0 JSON line.  The value
# it prints is NOT a scaling measurement (the ranks time-slice one GPU).
set -u
O=${1:-gpurun_out/share}
mkdir -p $O
for cfg in "2 c5 weak" "2 c4 strong" "2 c3a strong" "4 c2 weak"; do
  set -- $cfg
  SB200_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $1 --workload $2 --scaling $3 \
    --steps 2 --warmup 1 --no-cpu-baseline > $O/n$1_$2_$3.json 2> $O/n$1_$2_$3.err
  echo "n=$1 $2 $3 rc=$? $(head -c 300 $O/n$1_$2_$3.json)"
done

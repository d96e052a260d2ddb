# the bench's N-rank path (peer exchange with fused export, graph-captured steps) with 2 and 4 ranks on one GPU
for n in 2 4; do
  MESHPLAN_RANKS_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --config C1 --steps 5 --warmup 3 > gpurun_out/bench_shared_$n.log 2>&1; echo "shared n=$n rc=$?"; tail -1 gpurun_out/bench_shared_$n.log | cut -c1-700
done

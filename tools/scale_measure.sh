# Weak-scaling pass on one box: bench.py under torchrun at N=2 and N=4 (one process per GPU, NCCL).
mkdir -p gpurun_out
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo n=$n rc=$?
done

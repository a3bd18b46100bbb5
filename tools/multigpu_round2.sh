# Round-2 multi-GPU measurements (run as: gpurun --gpus 4 -- bash tools/multigpu_round2.sh)
python -m pytest tests/test_gpu_dp.py -q -rA > gpurun_out/dp4.log 2>&1; tail -9 gpurun_out/dp4.log
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n \
    bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  python -c "import json; d=json.load(open('gpurun_out/bench_n$n.json')); print($n, d['value'], d['ms_per_step'], d['e2e']['value'], d['stats']['global_images_per_s_median'])"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 \
  bench.py --gpus 4 --steps 20 --warmup 3 --lag 1 > gpurun_out/bench_n4_lag1.json 2> gpurun_out/bench_n4_lag1.err
python -c "import json; d=json.load(open('gpurun_out/bench_n4_lag1.json')); print('lag1', d['value'], d['ms_per_step'], d['e2e']['value'], d['last_loss'])"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 \
  bench.py --gpus 4 --steps 20 --warmup 3 --hierarchy 2x2 > gpurun_out/bench_n4_h22.json 2> gpurun_out/bench_n4_h22.err
python -c "import json; d=json.load(open('gpurun_out/bench_n4_h22.json')); print('2x2', d['value'], d['ms_per_step'], d['e2e']['value'])"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 \
  bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/bench_ref_n4.json 2> gpurun_out/bench_ref_n4.err
python -c "import json; d=json.load(open('gpurun_out/bench_ref_n4.json')); print('ref', d['value'], d['ms_per_step'], d['cpu_baseline']['cores'])"

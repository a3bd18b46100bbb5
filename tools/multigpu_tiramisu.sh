# Config 4 (Tiramisu, fp16) data-parallel: N=2 and N=4 (run as: gpurun --gpus 4 -- bash tools/multigpu_tiramisu.sh)
cd $GRAFT_REPO_ROOT
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n \
    bench.py --gpus $n --steps 20 --warmup 3 --variant tiramisu > gpurun_out/bench_tiramisu_n$n.json 2> gpurun_out/bench_tiramisu_n$n.err
  python -c "import json; d=json.load(open('gpurun_out/bench_tiramisu_n$n.json')); print($n, d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['precision'])"
done
python bench.py --variant tiramisu --steps 20 --no-cpu > gpurun_out/bench_tiramisu_n1.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_tiramisu_n1.json')); print(1, d['value'], d['ms_per_step'], d['e2e']['value'])"

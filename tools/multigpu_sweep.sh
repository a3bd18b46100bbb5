run() { tag=$1; shift; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --steps 20 --warmup 3 --no-cpu $BARGS > gpurun_out/mg_$tag.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/mg_$tag.json')); print('$tag', round(d['value'],1), round(d['ms_per_step'],3))"; }
BARGS="" run base X=1
BARGS="--bucket-mb 8" run b8 X=1
BARGS="--bucket-mb 64" run b64 X=1
BARGS="" run ch4 NCCL_MAX_NCHANNELS=4
BARGS="" run ch8 NCCL_MAX_NCHANNELS=8
BARGS="" run nvls0 NCCL_NVLS_ENABLE=0
BARGS="--lag 1" run lag1 X=1

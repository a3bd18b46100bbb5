cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_model.py tests/test_gpu_fp16.py -x -q 2>&1 | tail -2
for v in 1 2; do python bench.py --variant tiramisu --no-cpu --steps 20 > gpurun_out/t_$v.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/t_$v.json')); print('tira', round(d['value'],2), d['roofline']['all_convs']['frac'])"; done

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_prodshape.py tests/test_gpu_model.py tests/test_gpu_fp16.py tests/test_gpu_norm.py -x -q 2>&1 | tail -2
python tools/prof_rowtap.py fprop32 fprop96 wgrad32 wgrad64 wgrad96 dgrad32
python tools/prof_conv.py fprop_mn dgrad_m wgrad c1x1_fprop c1x1_dgrad stem_fprop_win stem_wgrad_win q_fprop s2b_dgrad
python bench.py --variant tiramisu --no-cpu --steps 20 > gpurun_out/t_new.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/t_new.json')); print('tira', round(d['value'],2), d['roofline']['all_convs']['frac'])"
for i in 1 2; do python bench.py --no-cpu --steps 30 > gpurun_out/m_new.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/m_new.json')); print('main', round(d['value'],2), round(d['stats']['rank_rate_median'],2), d['roofline']['frac'])"; done

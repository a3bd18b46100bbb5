cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_prodshape.py tests/test_gpu_model.py tests/test_gpu_fp16.py tests/test_gpu_norm.py -x -q 2>&1 | tail -3
for v in 3 5 3 5 3 5; do B2DL_ROWTAP_MINK=$v python bench.py --no-cpu --steps 30 > gpurun_out/mk_$v.json 2>/dev/null; python -c "import json; d=json.load(open(\"gpurun_out/mk_$v.json\")); print(\"bench $v\", round(d[\"value\"],2), round(d[\"stats\"][\"rank_rate_median\"],2))"; done

cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_norm.py tests/test_gpu_prodshape.py -x -q 2>&1 | tail -3
for v in 0 1; do echo "PW=$v"; B2DL_EPI_PW=$v python tools/prof_conv.py c1x1_dgrad c1x1_fprop q_fprop dgrad_m fprop_mn up_fprop; done
for v in 1 0 1 0; do B2DL_EPI_PW=$v python bench.py --no-cpu --steps 20 > gpurun_out/pw_$v.json 2>/dev/null; python -c "import json; d=json.load(open(\"gpurun_out/pw_$v.json\")); print(\"bench $v\", d[\"value\"], d[\"stats\"][\"rank_rate_median\"])"; done

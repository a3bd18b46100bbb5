cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py -k "rowtap or kblk" -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fp16.py tests/test_gpu_fp32.py -k "tiramisu or minidense or deeplab_config1" -x -q 2>&1 | tail -3
for v in 1 0; do echo "pairs=$v"; B2DL_ROWTAP_PAIRS=$v python tools/prof_rowtap.py fprop32 fprop64 fprop96 dgrad32 dgrad64; done
for v in 1 0 1 0; do B2DL_ROWTAP_PAIRS=$v python bench.py --variant tiramisu --no-cpu --steps 20 > gpurun_out/rp_$v.json 2>/dev/null; python -c "import json; d=json.load(open(\"gpurun_out/rp_$v.json\")); print(\"tira pairs=$v\", round(d[\"value\"],2), round(d[\"stats\"][\"rank_rate_median\"],2), d[\"roofline\"][\"all_convs\"][\"frac\"])"; done

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_norm.py tests/test_gpu_prodshape.py tests/test_gpu_model.py -x -q 2>&1 | tail -2
B2DL_EW16_NOPS=1 B2DL_EPI_SLOTS_16_2=2 ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/ll_old.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-graph > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/ll_new.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-graph > /dev/null 2>&1
for v in new old new old; do
  if [ $v = old ]; then e="B2DL_EW16_NOPS=1 B2DL_EPI_SLOTS_16_2=2"; else e="B2DL_X=1"; fi
  env $e python bench.py --no-cpu --steps 20 > gpurun_out/ew_$v.json 2>/dev/null; python -c "import json; d=json.load(open(\"gpurun_out/ew_$v.json\")); print(\"bench $v\", d[\"value\"], d[\"stats\"][\"rank_rate_median\"])"
done

# A/B of two builds on one box: ab_libs/libb2dl_base.so vs the in-tree libb2dl.so, alternating
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  for v in base new; do
    if [ $v = base ]; then e="B2DL_LIB_PATH=$PWD/ab_libs/libb2dl_base.so"; else e="B2DL_X=1"; fi
    env $e python bench.py --no-cpu --steps 20 ${AB_ARGS} > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['value'],2), round(d['stats']['rank_rate_median'],2))"
  done
done

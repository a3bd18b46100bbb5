# One-GPU measurement pass: bench (N=1), reference arm, memory-bound table, ncu launch list.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 300 python tools/prof_small.py --out gpurun_out/membound_kernels.txt > /dev/null 2>&1; echo small_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file gpurun_out/ncu_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-graph \
  > gpurun_out/ncu_bench.log 2>&1; echo ncu_rc=$?

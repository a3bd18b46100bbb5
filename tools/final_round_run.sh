set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --variant bn-bilinear --no-cpu > gpurun_out/final_bench_bn.json 2> gpurun_out/final_bench_bn.err; echo "bn rc=$?"
timeout 600 python bench.py --variant tiramisu --no-cpu > gpurun_out/final_bench_tira.json 2> gpurun_out/final_bench_tira.err; echo "tira rc=$?"

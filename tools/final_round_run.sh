# Final measurements of the round (run on one B200 box): GPU tests, smoke, bench lines, launch lists, ncu captures
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --variant bn-bilinear --no-cpu > gpurun_out/final_bench_bn.json 2> gpurun_out/final_bench_bn.err; echo "bn rc=$?"
timeout 600 python bench.py --variant tiramisu --no-cpu > gpurun_out/final_bench_tira.json 2> gpurun_out/final_bench_tira.err; echo "tira rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-graph > /dev/null 2>&1; echo "ll rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/final_tira_launches.csv python bench.py --variant tiramisu --steps 2 --warmup 1 --no-cpu --no-graph > /dev/null 2>&1; echo "tll rc=$?"
python tools/prof_conv.py fprop_mn dgrad_m wgrad up_dgrad > /dev/null && timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_ -c 4 -o gpurun_out/final_conv python tools/prof_conv.py fprop_mn dgrad_m wgrad up_dgrad > gpurun_out/final_conv.log 2>&1; echo "ncu rc=$?"
python tools/prof_rowtap.py fprop96 wgrad96 dgrad96 > gpurun_out/final_rowtap_events.txt 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:conv_rowtap -c 2 -o gpurun_out/final_rowtap python tools/prof_rowtap.py fprop96 wgrad96 > gpurun_out/final_rowtap.log 2>&1; echo "ncu rt rc=$?"
# summaries on the box; the full reports stay there (gpurun copies back at most 64 MiB)
python tools/ncu_summary.py gpurun_out/final_conv.ncu-rep > gpurun_out/final_conv_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/final_rowtap.ncu-rep > gpurun_out/final_rowtap_summary.txt 2>&1
ncu -i gpurun_out/final_conv.ncu-rep --page raw --csv > gpurun_out/final_conv_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out

mkdir -p gpurun_out; o=gpurun_out/epi_sweep.txt; : > $o
for cfg in "B2DL_EW16_NOPS=1" "B2DL_EPI_SLOTS_8_2=1" "B2DL_EPI_SLOTS_8_2=3" "B2DL_EW16_NOPS=2 B2DL_EPI_SLOTS_16_2=1" "B2DL_EW16_NOPS=2 B2DL_EPI_SLOTS_16_2=2"; do
  echo "== $cfg" >> $o
  env $cfg timeout 120 python tools/prof_conv.py c1x1_dgrad c1x1_fprop dgrad_m >> $o 2>&1
done

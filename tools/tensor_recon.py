"""Reconcile the tensor-pipe counters of a `ncu --set full` capture with executed MMA work.

    python tools/tensor_recon.py recon_raw.csv   (ncu -i <rep> --page raw --csv > recon_raw.csv)

For each conv kernel: UTCHMMA warp-instructions executed x FLOPs per instruction (M x N x K x 2
of the instruction shape: 256x256x16 for the CTA-pair fprop/dgrad, 128x256x16 for the wgrad)
vs the algorithmic 2*9*256*256*N*H*W, and the resulting FLOP rate vs the SM-clock peak
(148 SMs x 8192 dense bf16 FLOP/clk) next to ncu's tensor-pipe utilisation metrics."""
import csv
import sys

ALG = 2 * 9 * 256 * 256 * 2 * 1152 * 768
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]


def g(r, k):
    return float(r[hdr.index(k)].replace(",", ""))


print(f"algorithmic FLOPs per launch (3x3 256->256 at 2x1152x768): {ALG:.4e}")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    pair = "conv_fprop_kernel" in name and ", 2, " in name
    per_inst = (256 if pair else 128) * 256 * 16 * 2
    inst = g(r, "sm__inst_executed_pipe_tensor_subpipe_hmma.sum")
    dur = g(r, "gpu__time_duration.sum") * 1e-3          # ms -> s
    clk = g(r, "sm__cycles_elapsed.avg.per_second") * 1e9
    executed = inst * per_inst
    rate = executed / dur
    peak = 148 * 8192 * clk
    print(f"{name[:44]}")
    print(f"   UTCHMMA executed {inst:12.0f} x {per_inst} FLOP = {executed:.4e} (algorithmic x {executed / ALG:.4f})")
    print(f"   {dur * 1e3:.3f} ms at {clk / 1e9:.3f} GHz -> {rate / 1e12:.1f} TF/s = {100 * rate / peak:.1f} % of "
          f"148 x 8192 FLOP/clk at that clock")
    for k in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
              "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"):
        if k in hdr:
            print(f"   {k:100s} {g(r, k):6.1f} %")

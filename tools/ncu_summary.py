"""Key metrics + top stall reasons from an ncu report (development aid)."""
import csv
import subprocess
import sys

KEYS = [('gpu__time_duration.sum', 'duration'),
        ('TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed', 'tensor pipe %'),
        ('dram__bytes_read.sum', 'dram read'), ('dram__bytes_write.sum', 'dram write'),
        ('dram__throughput.avg.pct_of_peak_sustained_elapsed', 'dram %'),
        ('lts__throughput.avg.pct_of_peak_sustained_elapsed', 'L2 %'),
        ('l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'L1/smem %'),
        ('sm__inst_executed.avg.per_cycle_active', 'IPC'),
        ('sm__cycles_elapsed.avg.per_second', 'SM clock'), ('launch__registers_per_thread', 'regs'),
        ('launch__grid_size', 'grid')]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')]
    for r in rows[2:]:
        print('==', r[idx['Kernel Name']][:80])
        for k, name in KEYS:
            if k in idx:
                print(f"   {name:16s} {r[idx[k]]} {units[idx[k]]}")
        vals = sorted(((float(r[idx[h]] or 0), h) for h in stall), reverse=True)[:6]
        print('   stalls', ', '.join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for v, h in vals))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)

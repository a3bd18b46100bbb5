"""roofline_traffic.json (profiles/round<N>/) from an ncu --set full report of tools/prof_conv.py
fprop_mn dgrad_m wgrad (first three conv launches): DRAM bytes per launch of each pass's kernel
at the full-resolution 3x3x256 shape, next to its algorithmic operand bytes."""
import csv
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
PASSES = ["fprop", "dgrad", "wgrad"]
N, H, W, C = 2, 1152, 768, 256
# algorithmic bytes (bf16): fprop reads x + writes y (+ weights); dgrad reads dy + mask, writes dx;
# wgrad reads x + dy (fp32 partials counted separately by the reduction)
ALGO = {"fprop": 2 * N * H * W * C * 2, "dgrad": 3 * N * H * W * C * 2, "wgrad": 2 * N * H * W * C * 2}


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    res = {}
    for pas, r in zip(PASSES, rows[2:5]):
        rd = float(r[ix["dram__bytes_read.sum"]]) * SCALE.get(units[ix["dram__bytes_read.sum"]], 1)
        wr = float(r[ix["dram__bytes_write.sum"]]) * SCALE.get(units[ix["dram__bytes_write.sum"]], 1)
        res[pas] = {"launch": f"{r[ix['Kernel Name']][:60]} at 2x1152x768x256 3x3 (ncu --set full)",
                    "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                    "algorithmic_bytes_per_launch": ALGO[pas]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

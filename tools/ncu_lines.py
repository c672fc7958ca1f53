"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export per
CUDA source line: warp-stall samples, warp instructions, thread instructions
(SIMT efficiency = thread / (32 * warp instructions)).

  ncu -i rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main():
    fn = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    agg = {}
    cur_file, cur_line, hdr = None, None, None
    for row in csv.reader(open(fn)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = {h: i for i, h in enumerate(row)}
            continue
        if row[0] in ("Function Name",) or hdr is None:
            continue
        if row[0]:  # a source line row (aggregated over its SASS)
            cur_line = (cur_file, int(row[0]), row[1][:90])
            try:
                s = float(row[hdr["Warp Stall Sampling (All Samples)"]] or 0)
                wi = float(row[hdr["Instructions Executed"]] or 0)
                ti = float(row[hdr["Thread Instructions Executed"]] or 0)
            except (ValueError, KeyError):
                continue
            a = agg.setdefault(cur_line, [0.0, 0.0, 0.0])
            a[0] += s
            a[1] += wi
            a[2] += ti
    tot = [sum(v[i] for v in agg.values()) for i in range(3)]
    print(f"total samples {tot[0]:.0f} warp instr {tot[1]:.3e} SIMT eff {tot[2] / max(1, 32 * tot[1]):.3f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        eff = v[2] / max(1, 32 * v[1])
        print(f"{100 * v[0] / tot[0]:5.1f}% smp {100 * v[1] / tot[1]:5.1f}% inst eff {eff:4.2f}  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()

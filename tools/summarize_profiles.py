"""Summarise the outputs of tools/profile_round.sh (gpurun_out/prof_*) into
profiles/: the bench line, the kernel shares of the bench's launch list, the
per-kernel time and DRAM bytes of one 4,096-map U-Net forward (bench.py's
roofline.traffic) and the key metrics of the full captures.

  python tools/summarize_profiles.py [--round r01]
"""

from __future__ import annotations

import argparse
import collections
import csv
import glob
import json
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")


def ncu_rows(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    return hdr, [r for r in rows[h + 1:] if len(r) == len(hdr)]


def short(name):
    return name.split("(")[0].replace("void ", "")


def launches(rnd):
    hdr, rows = ncu_rows(os.path.join(OUT, "prof_launches.csv"))
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        k = short(r[iN])
        tot[k] += float(r[iV].replace(",", "")) / 1e3
        cnt[k] += 1
    s = sum(tot.values())
    path = os.path.join(PROF, f"{rnd}_launches_summary.csv")
    with open(path, "w") as f:
        f.write(f"# ncu launch list of `python bench.py --steps 1 --warmup 3 --no-graph` "
                f"({len(rows)} launches after 300 skipped)\n")
        f.write("# --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised -> "
                "compare shares\n")
        f.write("kernel,launches,total_us,share\n")
        for k, v in tot.most_common():
            f.write(f"{k},{cnt[k]},{v:.1f},{v / s:.3f}\n")
    return path


def network(rnd):
    hdr, rows = ncu_rows(os.path.join(OUT, "prof_net.csv"))
    iN, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iID = hdr.index("ID")
    per = collections.OrderedDict()
    for r in rows:
        d = per.setdefault(int(r[iID]), {"kernel": short(r[iN])})
        d[r[iM]] = float(r[iV].replace(",", ""))
    seq = list(per.values())
    # the last forward: from the last k_stack_to_nhwc to the end (torch copy /
    # reduction kernels of the checksum excluded)
    start = max(i for i, d in enumerate(seq) if "k_stack_to_nhwc" in d["kernel"])
    layers = []
    for d in seq[start:]:
        if not d["kernel"].startswith("drcb::"):
            continue
        layers.append({"kernel": d["kernel"], "us": round(d["gpu__time_duration.sum"] / 1e3, 1),
                       "dram_bytes": int(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"])})
    out = {"what": "U-Net forward of 4,096 maps (bench precision), DRAM bytes per kernel from ncu --metrics "
                   "dram__bytes_read.sum,dram__bytes_write.sum (--clock-control none, serialised)",
           "maps": 4096, "dram_bytes_total": sum(x["dram_bytes"] for x in layers),
           "kernel_us_total": round(sum(x["us"] for x in layers), 1), "layers": layers}
    path = os.path.join(PROF, f"{rnd}_network_traffic.json")
    json.dump(out, open(path, "w"), indent=1)
    return path


FULL_METRICS = [
    ("duration (gpu__time_duration.sum)", "gpu__time_duration.sum"),
    ("SM throughput % (sm__throughput.avg.pct_of_peak_sustained_elapsed)",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe active % (sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed)",
     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("issue active % (smsp__issue_active.avg.pct_of_peak_sustained_active)",
     "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("DRAM read (dram__bytes_read.sum)", "dram__bytes_read.sum"),
    ("DRAM write (dram__bytes_write.sum)", "dram__bytes_write.sum"),
    ("L2 bytes (lts__t_bytes.sum)", "lts__t_bytes.sum"),
    ("L2 hit % (lts__t_sector_hit_rate.pct)", "lts__t_sector_hit_rate.pct"),
    ("L1 hit % (l1tex__t_sector_hit_rate.pct)", "l1tex__t_sector_hit_rate.pct"),
    ("achieved occupancy % (sm__warps_active.avg.pct_of_peak_sustained_active)",
     "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("avg active threads / warp instr (smsp__thread_inst_executed_per_inst_executed.ratio)",
     "smsp__thread_inst_executed_per_inst_executed.ratio"),
    ("registers/thread (launch__registers_per_thread)", "launch__registers_per_thread"),
    ("grid (launch__grid_size)", "launch__grid_size"),
    ("block (launch__block_size)", "launch__block_size"),
]


def full(rnd):
    lines = [f"# {rnd} ncu --set full captures (bench.py config c3, eager steps, --clock-control none)",
             "", "Produced by tools/profile_round.sh; one launch per kernel after the warm-up.", ""]
    for rep in sorted(glob.glob(os.path.join(OUT, "prof_full_*.ncu-rep"))):
        name = os.path.basename(rep)[len("prof_full_"):-len(".ncu-rep")]
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout.splitlines()
        rows = list(csv.reader(raw))
        if len(rows) < 3:
            continue
        hdr, units, v = rows[0], rows[1], rows[2]
        lines.append(f"## {name}")
        lines.append(f"kernel: {v[hdr.index('Kernel Name')][:160]}")
        lines.append("")
        for label, key in FULL_METRICS:
            if key in hdr:
                lines.append(f"- {label}: {v[hdr.index(key)]} {units[hdr.index(key)]}")
        lines.append("")
    path = os.path.join(PROF, f"{rnd}_ncu_full_summary.md")
    open(path, "w").write("\n".join(lines) + "\n")
    return path


def traversal(rnd):
    """Memory traffic of the casting kernels (one launch = one frame's stage)
    from the full captures: L2 -> L1 bytes, L1 -> L2 write bytes, DRAM bytes."""
    out = {"what": "per-launch memory traffic of the ray-casting kernels (one 1024^2 c3 frame), "
                   "ncu --set full, --clock-control none",
           "kernels": {}}
    keys = {"us": "gpu__time_duration.sum", "l2_to_l1_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
            "l1_to_l2_write_bytes": "l1tex__m_l1tex2xbar_write_bytes.sum",
            "dram_read_bytes": "dram__bytes_read.sum", "dram_write_bytes": "dram__bytes_write.sum",
            "l1_hit_pct": "l1tex__t_sector_hit_rate.pct", "l2_hit_pct": "lts__t_sector_hit_rate.pct"}
    scale = {"us": 1e-3, "l2_to_l1_bytes": 1e9, "l1_to_l2_write_bytes": 1e9,
             "dram_read_bytes": 1e6, "dram_write_bytes": 1e6}
    for name in ("map_paths", "gbuffer_direct1"):
        rep = os.path.join(OUT, f"prof_full_{name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout.splitlines()
        rows = list(csv.reader(raw))
        hdr, units, v = rows[0], rows[1], rows[2]
        d = {}
        for k, m in keys.items():
            if m in hdr:
                val = float(v[hdr.index(m)].replace(",", ""))
                unit = units[hdr.index(m)]
                if k.endswith("bytes"):  # normalise to bytes
                    val *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                elif k == "us":
                    val *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(unit, 1)
                d[k] = val
        out["kernels"][name] = d
    path = os.path.join(PROF, f"{rnd}_traversal_traffic.json")
    json.dump(out, open(path, "w"), indent=1)
    return path


def train(rnd):
    """Kernel shares of one B = 4,096 tensor-core training step (the second of
    two: tools/train_time.py --warmup 1 --iters 1) with DRAM bytes."""
    hdr, rows = ncu_rows(os.path.join(OUT, "prof_train.csv"))
    iN, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = collections.OrderedDict()
    for r in rows:
        d = per.setdefault(int(r[iID]), {"kernel": short(r[iN])})
        d[r[iM]] = float(r[iV].replace(",", ""))
    seq = list(per.values())
    # the second step starts at its weight-prep launch (the first step also
    # runs the engine's one-time setup kernels)
    starts = [i for i, d in enumerate(seq) if "k_prep_weights" in d["kernel"]]
    seq = seq[starts[-1]:] if starts else seq[len(seq) // 2:]
    tot, cnt, dram = collections.Counter(), collections.Counter(), collections.Counter()
    for d in seq:
        k = d["kernel"]
        tot[k] += d.get("gpu__time_duration.sum", 0.0) / 1e3
        cnt[k] += 1
        dram[k] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    s = sum(tot.values())
    path = os.path.join(PROF, f"{rnd}_train_launches_summary.csv")
    with open(path, "w") as f:
        f.write("# ncu launch list of one bf16 tensor-core training step, B = 4,096 (the second of two), "
                "--clock-control none, serialised\n")
        f.write("kernel,launches,total_us,share,dram_gb\n")
        for k, v in tot.most_common():
            f.write(f"{k},{cnt[k]},{v:.1f},{v / s:.3f},{dram[k] / 1e9:.3f}\n")
    return path


def bench(rnd):
    for line in open(os.path.join(OUT, "prof_bench.log")):
        if line.startswith("{"):
            path = os.path.join(PROF, f"{rnd}_bench.json")
            json.dump(json.loads(line), open(path, "w"), indent=1)
            return path
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--out", default=None, help="output directory (default profiles/)")
    a = ap.parse_args()
    global PROF
    if a.out:
        PROF = a.out
        os.makedirs(PROF, exist_ok=True)
    for fn in (bench, launches, network, train, full, traversal):
        try:
            print(fn(a.round))
        except Exception as e:  # keep the others
            print(f"{fn.__name__}: {e!r}")


if __name__ == "__main__":
    main()

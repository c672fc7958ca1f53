#!/usr/bin/env bash
# Regenerate the round's profile evidence on a B200 (run under gpurun from the
# repo root), then `python tools/summarize_profiles.py` here writes profiles/.
#   1. bench.py line (no profiler)                       -> gpurun_out/prof_bench.log
#   2. ncu launch list of the bench (eager steps)         -> gpurun_out/prof_launches.csv
#   3. per-kernel time + DRAM bytes of one U-Net forward  -> gpurun_out/prof_net.csv
#   4. ncu --set full captures of the top kernels         -> gpurun_out/prof_full_*.ncu-rep
set -u
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-train --no-secondary --no-cpu-baseline --no-graph"
timeout 600 python bench.py > gpurun_out/prof_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 --csv \
  --log-file gpurun_out/prof_launches.csv $B > gpurun_out/prof_launches.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv python tools/net_time.py --iters 1 > gpurun_out/prof_net.csv 2>&1
full() {  # name, kernel regex, launches to skip
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$2" -s "$3" -c 1 -f \
    -o "gpurun_out/prof_full_$1" $B > "gpurun_out/prof_full_$1.log" 2>&1
}
full map_paths 'k_map_paths' 3
full gbuffer_direct1 'k_gbuffer_direct1' 3
full conv_pair 'k_conv_pair' 3
full conv_tc_dec3 'k_conv_tc' 34
full conv_rows_dec1 'k_conv_rows' 5   # 6 row-conv launches per frame: dec1.deconv2 is the 6th
full head_fused 'k_head_fused' 3
# summarise on the box (the ncu reports are large), keep two reports
python tools/summarize_profiles.py --out gpurun_out/profiles_new
for f in gpurun_out/prof_full_*.ncu-rep; do
  case "$f" in *map_paths*|*head_fused*) ;; *) rm -f "$f" ;; esac
done
ls -la gpurun_out gpurun_out/profiles_new

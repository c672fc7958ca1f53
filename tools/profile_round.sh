#!/usr/bin/env bash
# Regenerate the round's profile evidence on a B200 (run under gpurun from the
# repo root), then `python tools/summarize_profiles.py --round rNN` writes
# profiles/ (run here or on the box with --out).
#   1. bench.py line (no profiler)                        -> gpurun_out/prof_bench.log
#   2. ncu launch list of the bench (eager steps)          -> gpurun_out/prof_launches.csv
#   3. per-kernel time + DRAM bytes of one U-Net forward   -> gpurun_out/prof_net.csv
#   4. ncu launch list of one tensor-core training step    -> gpurun_out/prof_train.csv
#   5. ncu --set full captures of the top kernels          -> gpurun_out/prof_full_*.ncu-rep
set -u
mkdir -p gpurun_out
NET=${NET:-fp16}
B="python bench.py --steps 1 --warmup 3 --no-train --no-secondary --no-cpu-baseline --no-graph"
T="python tools/train_time.py --batch 4096 --warmup 1 --iters 1"
timeout 900 python bench.py > gpurun_out/prof_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 400 --csv \
  --log-file gpurun_out/prof_launches.csv $B > gpurun_out/prof_launches.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv python tools/net_time.py --iters 1 --mode $NET > gpurun_out/prof_net.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/prof_train.csv $T > gpurun_out/prof_train.out 2>&1
full() {  # name, kernel regex, launches to skip, command
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$2" -s "$3" -c 1 -f \
    -o "gpurun_out/prof_full_$1" $4 > "gpurun_out/prof_full_$1.log" 2>&1
}
full map_paths 'k_map_paths' 3 "$B"
full gbuffer_direct1 'k_gbuffer_direct1' 3 "$B"
full conv_pair 'k_conv_pair' 3 "$B"
full conv_tc_dec3 'k_conv_tc' 34 "$B"
full conv_rows_dec1 'k_conv_rows' 5 "$B"   # 6 row-conv launches per frame: dec1.deconv2 is the 6th
full head_fused 'k_head_fused' 3 "$B"
full interp 'k_interp' 3 "$B"   # the gather-bound elementwise stages (issue, not HBM)
full shade 'k_shade' 3 "$B"
full train_wgrad_dxn 'k_wgrad_dxn' 12 "$T"  # second step's first (head.deconv2)
full train_wgrad_taps '^k_wgrad$' 6 "$T"
full train_bnb_apply 'k_bnb_apply' 17 "$T"
# summarise on the box (the ncu reports are large), keep two reports
python tools/summarize_profiles.py --round "${ROUND:-r02}" --out gpurun_out/profiles_new
for f in gpurun_out/prof_full_*.ncu-rep; do
  case "$f" in *map_paths*|*wgrad_dxn*) ;; *) rm -f "$f" ;; esac
done
ls -la gpurun_out gpurun_out/profiles_new

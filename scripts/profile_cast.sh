# ncu evidence for the config-3 batched cast (run through gpurun; outputs in gpurun_out/):
#   launches.csv       launch list of a short bench.py run (per-launch durations, serialised)
#   prof_step_warm     --set full of every launch of one 100M-query step, warm L2 (--cache-control none)
#   prof_step_cold     the same with caches flushed per kernel (ncu default)
#   prof_p1 / prof_w0  single-launch reports (warm) of phase 1 and window pass 0, for the
#                      stall breakdown and SASS hot spots (summarize_ncu.py per kernel)
set -x
K='regex:k_cast_defer|k_walk_pass|k_walk_last|k_cast_near'
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --cpu-sample 1000000 --pf-iterations 0 --no-extra > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k "$K" -s 36 -c 12 \
  -o gpurun_out/prof_step_warm -f python scripts/cast_timing.py > gpurun_out/ncu_warm.log 2>&1
ncu --set full --clock-control none --import-source on -k "$K" -s 36 -c 12 \
  -o gpurun_out/prof_step_cold -f python scripts/cast_timing.py > gpurun_out/ncu_cold.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_cast_defer_p1 -s 6 -c 1 \
  -o gpurun_out/prof_p1 -f python scripts/cast_timing.py > gpurun_out/ncu_p1.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_walk_pass -s 24 -c 1 \
  -o gpurun_out/prof_w0 -f python scripts/cast_timing.py > gpurun_out/ncu_w0.log 2>&1
echo done
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_walk_last -s 6 -c 1 \
  -o gpurun_out/prof_last -f python scripts/cast_timing.py > gpurun_out/ncu_last.log 2>&1
echo done

# ncu evidence for the config-5 edit kernels (run through gpurun after round_measure.sh; outputs in gpurun_out/)
bash scripts/round_measure.sh
ncu --set full --clock-control none --cache-control none --import-source on -k regex:'k_merge_touched|k_bucket_plan|k_flags_bucket' -s 60 -c 3 -o gpurun_out/prof_edit -f timeout 300 python scripts/edit_timing.py 30 > gpurun_out/ncu_edit.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:'k_merge_touched' -s 20 -c 1 -o gpurun_out/prof_merge -f timeout 300 python scripts/edit_timing.py 30 > gpurun_out/ncu_merge.log 2>&1
echo done

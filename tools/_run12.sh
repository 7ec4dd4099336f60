python tools/sweep.py city_batch '{"window": [1200, 2400, 600]}' --reps 3 > gpurun_out/r02_sweep_12.jsonl 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_query_cta -s 1 -c 1 -o gpurun_out/r02_batch_v2 python tools/profile_target.py city_batch --reps 2 > gpurun_out/r02_ncu_batch_v2.log 2>&1

python tools/sweep.py metro_batch '{"cluster_dir": ["auto", "compact"]}' --reps 3 >> gpurun_out/r02_dir_metro.jsonl
python tools/sweep.py single:metro '{"cluster_dir": ["auto", "compact"]}' --reps 5 >> gpurun_out/r02_dir_metro.jsonl
python tools/sweep.py single:country '{"cluster_dir": ["auto", "compact"]}' --reps 3 >> gpurun_out/r02_dir_metro.jsonl
ncu --set full --import-source on --clock-control none -k regex:k_query_cta -s 1 -c 1 -o gpurun_out/r02_batch_v1 python tools/profile_target.py city_batch --reps 2 > gpurun_out/r02_ncu_batch_v1.log 2>&1

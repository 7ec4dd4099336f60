python -m pytest tests -x -q -m gpu -k "metro_batched or grouped or goal or two_streams or multi_device" > gpurun_out/pytest_r02_15.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02_15.log
python bench.py --workload metro_batch --steps 5 --warmup 3 --latency "" > gpurun_out/bench_r02_15_metro_batch.json 2> gpurun_out/bench_r02_15_metro_batch.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:k_query_groups -c 2 --csv python tools/profile_target.py metro_batch --reps 2 > gpurun_out/r02_ncu_groups_flat.csv 2>&1

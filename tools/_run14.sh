for v in cur2 groupsflat cur2 groupsflat; do python tools/sweep.py metro_batch '{}' --reps 3 --lib ab/libeat_$v.so >> gpurun_out/r02_groupsflat.jsonl 2>>gpurun_out/r02_groupsflat.err; done
for v in cur2 groupsflat; do python tools/sweep.py metro_batch '{"window": [600, 2400, 7200]}' --reps 3 --lib ab/libeat_$v.so >> gpurun_out/r02_groupsflat.jsonl 2>>gpurun_out/r02_groupsflat.err; done

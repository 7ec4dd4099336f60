for r in 1 2 3; do for v in cur mopt lazyr1; do python tools/ab_lib.py ab/libeat_$v.so 3 >> gpurun_out/ab_r02_7.jsonl 2>>gpurun_out/ab_r02_7.err; done; done
python tools/sweep.py metro_batch '{}' --reps 3 --lib ab/libeat_mopt.so >> gpurun_out/ab_r02_7m.jsonl
python tools/sweep.py metro_batch '{}' --reps 3 --lib ab/libeat_lazyr1.so >> gpurun_out/ab_r02_7m.jsonl
python tools/sweep.py single:metro '{}' --reps 5 --lib ab/libeat_mopt.so >> gpurun_out/ab_r02_7m.jsonl
python tools/sweep.py single:metro '{}' --reps 5 --lib ab/libeat_lazyr1.so >> gpurun_out/ab_r02_7m.jsonl

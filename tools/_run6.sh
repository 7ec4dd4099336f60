for r in 1 2; do for v in cur mopt; do python tools/ab_lib.py ab/libeat_$v.so 3 >> gpurun_out/ab_r02_6.jsonl 2>>gpurun_out/ab_r02_6.err; done; done
python -m pytest tests -x -q -m gpu -k "selftest or tiny or random_small or window or arr16 or goal or subtrips or city_batch or lookup" > gpurun_out/pytest_r02_6.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02_6.log

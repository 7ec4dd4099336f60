for r in 1 2 3; do for v in early owner; do python tools/ab_lib.py ab/libeat_$v.so 3 >> gpurun_out/ab_r02_10.jsonl 2>>gpurun_out/ab_r02_10.err; done; done
python -m pytest tests -x -q -m gpu -k "selftest or tiny or random_small or window or goal or city_batch or arr16 or subtrips or invalid" > gpurun_out/pytest_r02_10.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02_10.log

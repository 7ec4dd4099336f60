for r in 1 2 3; do for v in mopt nodense early; do python tools/ab_lib.py ab/libeat_$v.so 3 >> gpurun_out/ab_r02_9.jsonl 2>>gpurun_out/ab_r02_9.err; done; done
python -m pytest tests -x -q -m gpu -k "selftest or tiny_batched or random_small or window or goal or city_batch" > gpurun_out/pytest_r02_9.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02_9.log

python tools/e2e_modes.py > gpurun_out/r02_e2e_modes.jsonl 2>&1
python -m pytest tests -x -q -m gpu -k "city_batch or tiny_batched or arr16 or two_streams" > gpurun_out/pytest_r02_13.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r02_13.log

for r in 1 2 3; do for v in early owner bsearch_shfl smem_lds bsearch_lds; do python tools/ab_lib.py ab/libeat_$v.so 3 >> gpurun_out/ab_r02_11.jsonl 2>>gpurun_out/ab_r02_11.err; done; done

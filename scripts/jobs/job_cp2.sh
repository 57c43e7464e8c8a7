#!/bin/bash
out=gpurun_out/${OUT:-cp2}; mkdir -p $out
timeout 600 python scripts/dbg/dbg_cp_tasks.py rmat24 > $out/dbg_cp_tasks.txt 2>&1
timeout 600 python scripts/ab_cp.py rmat24 > $out/ab_cp.jsonl 2>> $out/err.txt
BBTC_FORCE_CP=1 timeout 600 python scripts/ab_cp.py rmat24 >> $out/ab_cp.jsonl 2>> $out/err.txt
timeout 1800 python -m pytest tests -m gpu -q -x -k "stream or out_of_core or device_input or full_size or dense_and_sparse or auto_p" > $out/tests.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-ncu > $out/bench_rmat24.json 2> $out/bench.err
echo done > $out/done.txt

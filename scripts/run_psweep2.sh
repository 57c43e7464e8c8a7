#!/bin/bash
# p-sweeps with bitmap batches in the list kernel
out=gpurun_out/r1t; mkdir -p $out
timeout 600 python scripts/p_sweep.py rmat24 12 16 20 24 28 32 >> $out/psweep_rmat24.jsonl 2>&1
timeout 600 python scripts/p_sweep.py orkut 4 6 8 12 16 >> $out/psweep_orkut.jsonl 2>&1
timeout 900 python scripts/p_sweep.py friendster 4 8 16 24 32 >> $out/psweep_friendster.jsonl 2>&1
echo done

#!/bin/bash
# f3/f4 measurements + the A/B of the streamed column source.
out=gpurun_out/${OUT:-f34}; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "hybrid or refinement" > $out/tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 600 python scripts/ab_cp.py rmat24 > $out/ab_cp.jsonl 2>> $out/err.txt
BBTC_FORCE_CP=1 timeout 600 python scripts/ab_cp.py rmat24 >> $out/ab_cp.jsonl 2>> $out/err.txt; echo "ab rc=$?" >> $out/steps.txt
timeout 1200 python scripts/hybrid_sweep.py karate rmat16 orkut > $out/hybrid.jsonl 2>> $out/err.txt; echo "hybrid rc=$?" >> $out/steps.txt
timeout 1500 python scripts/study_f4.py psweep rmat24 4 8 12 16 24 32 > $out/psweep_rmat24.jsonl 2>> $out/err.txt; echo "psweep rc=$?" >> $out/steps.txt
timeout 1200 python scripts/study_f4.py psweep orkut 4 8 12 16 32 > $out/psweep_orkut.jsonl 2>> $out/err.txt
timeout 1200 python scripts/study_f4.py estim rmat24 16 > $out/estim_rmat24.jsonl 2>> $out/err.txt; echo "estim rc=$?" >> $out/steps.txt
timeout 1200 python scripts/study_f4.py estim orkut 16 > $out/estim_orkut.jsonl 2>> $out/err.txt
timeout 1500 python scripts/study_f4.py estim friendster 16 > $out/estim_friendster.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt

#!/bin/bash
# Per-task device times (bbtc_task_times) at the bench configs, for the multi-GPU balance study.
out=gpurun_out/${OUT:-r02cc}; mkdir -p $out
timeout 1200 python scripts/study_f4.py estim rmat24 10 > $out/estim_rmat24_p10.jsonl 2>> $out/err.txt
timeout 1200 python scripts/study_f4.py estim orkut 8 > $out/estim_orkut_p8.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt

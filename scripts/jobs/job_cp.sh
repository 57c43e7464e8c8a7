#!/bin/bash
out=gpurun_out/${OUT:-cp}; mkdir -p $out
for mode in plain cp; do
  env=""; [ $mode = cp ] && export BBTC_FORCE_CP=1 || unset BBTC_FORCE_CP
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_count$' -s 5 -c 1 \
    -o $out/prof_$mode python scripts/ab_cp.py rmat24 > $out/ncu_$mode.log 2>&1
  ncu -i $out/prof_$mode.ncu-rep --page source --csv --print-source cuda > $out/src_$mode.csv 2>/dev/null
  ncu -i $out/prof_$mode.ncu-rep --page raw --csv > $out/raw_$mode.csv 2>/dev/null
done
unset BBTC_FORCE_CP
timeout 900 python scripts/study_f4.py estim rmat24 16 > $out/estim_rmat24.jsonl 2>> $out/err.txt
timeout 900 python scripts/study_f4.py estim orkut 16 > $out/estim_orkut.jsonl 2>> $out/err.txt
timeout 900 python scripts/study_f4.py estim friendster 16 > $out/estim_friendster.jsonl 2>> $out/err.txt
echo done > $out/done.txt

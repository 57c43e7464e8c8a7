#!/bin/bash
# Full check at HEAD: GPU tests, default bench (with in-run ncu traffic and the full
# oracle baseline), reference arm, launch list, estimator study, sanitizer reruns.
out=gpurun_out/${OUT:-r02e}; mkdir -p $out
timeout 900 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err; echo "bench rc=$?" >> $out/steps.txt
timeout 2400 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/ref_rmat24.json 2> $out/ref.err; echo "ref rc=$?" >> $out/steps.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches_rmat24.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ncu --e2e-steps 1 > $out/launches.log 2>&1; echo "launches rc=$?" >> $out/steps.txt
timeout 900 python scripts/study_f4.py estim rmat24 16 > $out/estim_rmat24.jsonl 2>> $out/err.txt
timeout 900 python scripts/study_f4.py estim orkut 16 > $out/estim_orkut.jsonl 2>> $out/err.txt
timeout 900 python scripts/study_f4.py estim friendster 16 > $out/estim_friendster.jsonl 2>> $out/err.txt; echo "estim rc=$?" >> $out/steps.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tests/gpu_child.py rmat:16:16:9 7 \
    resident,ranks3,streamed,sranks3,ooc25,ooc50,stage rowmajor > $out/san_$tool.rowmajor.log 2>&1
  echo "san $tool rowmajor rc=$?" >> $out/steps.txt
  timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tests/gpu_child.py rmat:16:16:9 7 \
    resident,ranks3,streamed,sranks3,ooc25,ooc50,stage > $out/san_$tool.col.log 2>&1
  echo "san $tool col rc=$?" >> $out/steps.txt
done
echo done >> $out/steps.txt

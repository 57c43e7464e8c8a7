#!/bin/bash
# One GPU box session: STEPS (comma list) of
#   smoke | bench[:config] | ref[:config] | tests[:-k expr] | slow | sanitize | ncu:<config>[:kernel regex]
# Outputs under gpurun_out/$OUT.
out=gpurun_out/${OUT:-job}; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used,memory.total --format=csv > $out/gpu.txt 2>&1
IFS=',' read -ra S <<< "${STEPS:-smoke,bench,tests}"
for st in "${S[@]}"; do
  kind=${st%%:*}; arg=${st#*:}; [ "$arg" = "$st" ] && arg=""
  case $kind in
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1 ;;
    bench) c=${arg:-rmat24}; timeout 1500 python bench.py --config $c $BENCH_ARGS > $out/bench_$c.json 2> $out/bench_$c.err ;;
    ref) c=${arg:-rmat24}; timeout 1500 python bench.py --impl reference --config $c --steps ${REF_STEPS:-20} --warmup ${REF_WARMUP:-5} > $out/ref_$c.json 2> $out/ref_$c.err ;;
    tests) if [ -n "$arg" ]; then timeout 2400 python -m pytest tests -m gpu -q -x -k "$arg" > $out/gpu_tests.log 2>&1;
           else timeout 2400 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1; fi ;;
    sanitize) OUT=${OUT:-job}/sanitize bash scripts/sanitize.sh ;;
    ncu) c=${arg%%:*}; k=${arg#*:}; [ "$k" = "$arg" ] && k=k_count
         timeout 1800 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-2} -c 1 \
           -o $out/prof_${c}_$k python scripts/profile_count.py $c > $out/ncu_${c}_$k.log 2>&1
         ncu -i $out/prof_${c}_$k.ncu-rep --page raw --csv > $out/ncu_${c}_$k.raw.csv 2>/dev/null
         ncu -i $out/prof_${c}_$k.ncu-rep --page source --csv --print-source cuda > $out/ncu_${c}_$k.src.csv 2>/dev/null ;;
    launches) c=${arg:-rmat24}; timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
           --log-file $out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-ncu --e2e-steps 1 > $out/launches_$c.log 2>&1 ;;
  esac
  echo "$st rc=$?" >> $out/steps.txt
done
echo done >> $out/steps.txt

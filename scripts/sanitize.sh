#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over every count mode on karate and
# R-MAT 16: resident (list + bit-row kernels), a rank split, streamed, streamed ranks,
# out of core at 25/50%, staged; column-major and row-major walks.  Logs to $out.
out=gpurun_out/${OUT:-sanitize}; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
modes=resident,ranks3,streamed,sranks3,ooc25,ooc50,stage
for tool in memcheck racecheck synccheck; do
  for spec in "karate:1 2" "rmat:16:16:9 7" "rmat:16:16:9 16"; do
    set -- $spec
    for walk in col rowmajor; do
      tag=$tool.$(echo $1 | tr ':' '_').p$2.$walk
      extra=""; [ $walk = rowmajor ] && extra=rowmajor
      timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
        python tests/gpu_child.py $1 $2 $modes $extra > $out/$tag.log 2>&1
      echo "$tag rc=$?" >> $out/summary.txt
    done
  done
done
echo done >> $out/summary.txt

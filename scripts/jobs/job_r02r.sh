#!/bin/bash
# Probe slots: parity tests + A/B; band crash localisation over kernel variants.
out=gpurun_out/${OUT:-r02r}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "probe_slots" > $out/test_slots.log 2>&1; echo "slots tests rc=$?" >> $out/steps.txt
for v in nopipe nolw nobm hint; do
  BBTC_SYNC_CHECK=1 BBTC_LIB=$PWD/build_ab/$v/libbbtc.so BBTC_BANDS=1 BBTC_BAND_BYTES=65536 timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/bands_$v.log 2>&1; echo "bands $v rc=$?" >> $out/steps.txt
done
timeout 3000 python scripts/ab_variants.py friendster,orkut,rmat24:10 paper_2009_12457_b200/libbbtc.so "env:BBTC_SLOTS=0" "env:BBTC_SLOT_MAX_DEG=16" > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt

#!/bin/bash
out=gpurun_out/r1z5; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or rmat16 or many_parts or random_graphs or karate or blocks_round or streaming or out_of_core" > $out/gpu_tests.log 2>&1
for x in 1 2; do
for pk in 1 0; do
  for cfg in rmat24 orkut friendster; do
    BBTC_TRACE=1 BBTC_PACKED_TRANSPOSE=$pk timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") 2> $out/trace_${cfg}_$pk.err | sed "s/^{/{\"v\": \"packed$pk\", /" >> $out/ab.jsonl
  done
done
done

timeout 600 python scripts/stream_probe.py rmat24 2>&1 | grep "\"copy_streams\": 2" >> gpurun_out/r1z5/stream_rmat24.jsonl
echo done

timeout 900 python scripts/p_sweep.py friendster 1 2 3 4 > gpurun_out/ps2_friendster.jsonl 2> gpurun_out/ps2.err
timeout 600 python scripts/p_sweep.py orkut 1 2 4 8 > gpurun_out/ps2_orkut.jsonl 2>> gpurun_out/ps2.err
timeout 600 python scripts/p_sweep.py rmat24 4 8 16 > gpurun_out/ps2_rmat24.jsonl 2>> gpurun_out/ps2.err
echo done

set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "dense or karate or rmat16_p_grid or random_graphs or degenerate or streaming or many_parts or out_of_core" > gpurun_out/dense_tests.log 2>&1
tail -3 gpurun_out/dense_tests.log
timeout 600 python scripts/dense_sweep.py rmat24 > gpurun_out/dense_rmat24.jsonl 2> gpurun_out/dense_rmat24.err
timeout 300 python scripts/dense_sweep.py rmat16 16 > gpurun_out/dense_rmat16.jsonl 2>> gpurun_out/dense_rmat24.err
timeout 300 python scripts/dense_sweep.py orkut 8 0,2048 > gpurun_out/dense_orkut.jsonl 2>> gpurun_out/dense_rmat24.err
echo done

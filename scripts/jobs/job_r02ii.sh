#!/bin/bash
# HEAD final (after the shard-block zeroing): GPU tests, smoke, rmat24 bench, the sharded bench path with 4 ranks (gloo, one GPU).
out=gpurun_out/${OUT:-r02ii}; mkdir -p $out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/steps.txt
timeout 2700 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > $out/bench_rmat24.json 2> $out/bench_rmat24.err; echo "bench rc=$?" >> $out/steps.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29534 \
  bench.py --gpus 4 --config orkut --steps 3 --warmup 3 --e2e-steps 1 > $out/bench_orkut_n4.json 2> $out/bench_orkut_n4.err; echo "n4 rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt

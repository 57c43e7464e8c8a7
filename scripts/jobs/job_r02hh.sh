#!/bin/bash
# The bench's N=2 sharded path on rmat16 (the failing GPU test): before / after zeroing unowned shard blocks.
out=gpurun_out/${OUT:-r02hh}; mkdir -p $out
BBTC_LIB=$PWD/build_ab/prefix/libbbtc.so timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29544 \
  bench.py --gpus 2 --config rmat16 --steps 3 --warmup 3 --e2e-steps 1 > $out/before.json 2> $out/before.err; echo "before rc=$?" >> $out/steps.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29545 \
  bench.py --gpus 2 --config rmat16 --steps 3 --warmup 3 --e2e-steps 1 > $out/after.json 2> $out/after.err; echo "after rc=$?" >> $out/steps.txt
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu > $out/tests_multi.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt

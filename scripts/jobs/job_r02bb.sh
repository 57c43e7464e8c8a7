#!/bin/bash
# The bench's N>1 (sharded) path at full rmat24 / orkut scale: 4 and 8 ranks sharing the one GPU (gloo) —
# a functional check of the routing / forwarding / all-reduce logic the SCALE run uses (timings not meaningful).
out=gpurun_out/${OUT:-r02bb}; mkdir -p $out
for n in 4 8; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=2950$n \
    bench.py --gpus $n --config orkut --steps 3 --warmup 3 --e2e-steps 1 > $out/bench_orkut_n$n.json 2> $out/bench_orkut_n$n.err
  echo "orkut n=$n rc=$?" >> $out/steps.txt
done
timeout 2000 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29514 \
  bench.py --gpus 4 --config rmat24 --steps 3 --warmup 3 --e2e-steps 1 > $out/bench_rmat24_n4.json 2> $out/bench_rmat24_n4.err
echo "rmat24 n=4 rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt

out=gpurun_out/dbg1; mkdir -p $out
timeout 120 python tests/gpu_child.py karate:1 2 streamed > $out/karate.log 2>&1; echo "karate rc=$?" >> $out/s.txt
timeout 120 python tests/gpu_child.py rmat:12:16:1 4 streamed,ooc50 > $out/r12.log 2>&1; echo "r12 rc=$?" >> $out/s.txt
timeout 120 env CUDA_LAUNCH_BLOCKING=1 python tests/gpu_child.py rmat:12:16:1 4 streamed > $out/r12b.log 2>&1; echo "r12b rc=$?" >> $out/s.txt
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 python tests/gpu_child.py rmat:12:16:1 4 streamed > $out/r12m.log 2>&1; echo "r12m rc=$?" >> $out/s.txt
timeout 120 python tests/gpu_child.py rmat:16:16:9 7 streamed > $out/r16.log 2>&1; echo "r16 rc=$?" >> $out/s.txt

#!/bin/bash
out=gpurun_out/dbg; mkdir -p $out
BBTC_NO_RP_ZERO=1 timeout 300 python scripts/stream_probe.py rmat16 > $out/s_norpz16.jsonl 2> $out/s_norpz16.err
timeout 300 python scripts/stream_probe.py rmat16 > $out/s_def16.jsonl 2> $out/s_def16.err
BBTC_NO_RP_ZERO=1 timeout 300 python scripts/stream_probe.py rmat24 > $out/s_norpz.jsonl 2> $out/s_norpz.err
BBTC_PACKED_TRANSPOSE=0 timeout 300 python scripts/stream_probe.py rmat24 > $out/s_nopack.jsonl 2> $out/s_nopack.err
echo done

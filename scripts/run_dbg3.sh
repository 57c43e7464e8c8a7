#!/bin/bash
out=gpurun_out/dbg3; mkdir -p $out
BBTC_LIB=abl/libbbtc_pf1.so timeout 600 python scripts/stream_probe.py friendster 2>&1 | grep '"copy_streams": 2' | sed 's/^{/{"v": "pf1", /' >> $out/s.jsonl
BBTC_ITEMS_PER_SLOT=24 timeout 600 python scripts/stream_probe.py friendster 2>&1 | grep '"copy_streams": 2' | sed 's/^{/{"v": "ips24", /' >> $out/s.jsonl
BBTC_ITEMS_PER_SLOT=96 timeout 600 python scripts/stream_probe.py friendster 2>&1 | grep '"copy_streams": 2' | sed 's/^{/{"v": "ips96", /' >> $out/s.jsonl
BBTC_STREAM_ORDER=exec timeout 600 python scripts/stream_probe.py friendster 2>&1 | grep '"copy_streams": 2' | sed 's/^{/{"v": "exec", /' >> $out/s.jsonl
echo done

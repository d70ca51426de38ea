#!/bin/bash
mkdir -p gpurun_out/r02
export MMA_SPIN_TIMEOUT_MS=8000
timeout 900 ncu --clock-control none --set full --import-source on --metrics nvlrx__bytes.sum,nvltx__bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum \
    -k regex:relay_pull -c 4 -f -o gpurun_out/prof_relay_proto_pull python scripts/ncu_relay_protocol.py > gpurun_out/ncu_relay_proto_pull.log 2>&1; echo "pull rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02/g_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02/g_all.log
tail -15 gpurun_out/r02/g_all.log

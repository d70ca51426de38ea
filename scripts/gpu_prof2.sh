#!/bin/bash
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 900 $NCU --set full --import-source on -k regex:zc_ -c 1 -f -o gpurun_out/prof_zc_h2d \
    python scripts/ncu_one_kernel.py --dir h2d > gpurun_out/ncu_zc_h2d.log 2>&1; echo "zc h2d rc=$?"
timeout 900 $NCU --replay-mode application -k regex:zc_ -c 1 -f -o gpurun_out/prof_zc_d2h \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,lts__t_bytes.sum \
    python scripts/ncu_one_kernel.py --dir d2h > gpurun_out/ncu_zc_d2h.log 2>&1; echo "zc d2h rc=$?"
timeout 900 $NCU --set full --import-source on --metrics nvlrx__bytes.sum,nvltx__bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum \
    -k regex:relay -c 8 -f -o gpurun_out/prof_relay_proto python scripts/ncu_relay_protocol.py > gpurun_out/ncu_relay_proto.log 2>&1; echo "proto rc=$?"

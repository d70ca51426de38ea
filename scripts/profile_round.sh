#!/bin/bash
# ncu evidence for the current code on one B200 (run under gpurun); reports land in gpurun_out/.
# Read them here with scripts/ncu_summarize.py, which writes profiles/ncu_summary.json and the
# per-kernel CSVs under profiles/.
#   1. launch list of the bench (per-launch gpu__time_duration, cold, serialised)
#   2. --set full of the zero-copy gather (config-3 KV fetch, H2D), one launch
#   3. DRAM / PCIe counters of the zero-copy scatter (config-3 KV offload, D2H); host-writing
#      kernels return nan under kernel replay, so application replay with a metric list
#   4. --set full of the relay pull / pack kernels alone (scripts/probe/probe_relay ncu:
#      7 rings x 8 CTAs, hop 1 complete, slots in local HBM)
#   5. --set full + NVLink counters of the relay pack and pull kernels in the engine's real
#      protocol (scripts/ncu_relay_protocol.py: waves of S chunks through mma_memcpy_*;
#      loopback rings on one GPU, peer rings with --peers on a multi-GPU box)
mkdir -p gpurun_out
NCU="ncu --clock-control none"
[ -x scripts/probe/probe_relay ] || nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -I include scripts/probe/probe_relay.cu -o scripts/probe/probe_relay
timeout 900 $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --quick --no-verify --modes zc,zc > gpurun_out/ncu_launch_bench.log 2>&1
echo "launch list rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:zc_ -c 1 -f -o gpurun_out/prof_zc_h2d \
    python scripts/ncu_one_kernel.py --dir h2d > gpurun_out/ncu_zc_h2d.log 2>&1
echo "zc h2d rc=$?"
timeout 900 $NCU --replay-mode application -k regex:zc_ -c 1 -f -o gpurun_out/prof_zc_d2h \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,lts__t_bytes.sum \
    python scripts/ncu_one_kernel.py --dir d2h > gpurun_out/ncu_zc_d2h.log 2>&1
echo "zc d2h rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:relay -c 2 -f -o gpurun_out/prof_relay \
    ./scripts/probe/probe_relay ncu > gpurun_out/ncu_relay.log 2>&1
echo "relay rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:relay -s 2 -c 2 -f -o gpurun_out/prof_relay_seg \
    ./scripts/probe/probe_relay ncu > gpurun_out/ncu_relay_seg.log 2>&1
echo "relay seg rc=$?"
[ -n "$PROFILE_ONLY_PROTO" ] && exit 0
PEERS=""; [ "$(nvidia-smi -L | wc -l)" -gt 1 ] && PEERS="--peers"
timeout 900 $NCU --set full --import-source on --metrics nvlrx__bytes.sum,nvltx__bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum \
    -k regex:relay_pack -c 4 -f -o gpurun_out/prof_relay_proto python scripts/ncu_relay_protocol.py $PEERS > gpurun_out/ncu_relay_proto.log 2>&1
echo "relay protocol (pack) rc=$?"
timeout 900 $NCU --set full --import-source on --metrics nvlrx__bytes.sum,nvltx__bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum \
    -k regex:relay_pull -c 4 -f -o gpurun_out/prof_relay_proto_pull python scripts/ncu_relay_protocol.py $PEERS > gpurun_out/ncu_relay_proto_pull.log 2>&1
echo "relay protocol (pull) rc=$?"

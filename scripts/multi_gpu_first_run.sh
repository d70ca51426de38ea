#!/bin/bash
# First run on a box with several GPUs: peer parity before any number, then
# the scaling line, the ring sweeps over real NVLink and ncu of the relay kernels reading peer
# memory. Everything lands in gpurun_out/mgpu/.
set -u
out=gpurun_out/mgpu; mkdir -p $out
export MMA_SPIN_TIMEOUT_MS=${MMA_SPIN_TIMEOUT_MS:-8000}
n=$(nvidia-smi -L | wc -l)
bash scripts/probe_box.sh > /dev/null 2>&1; cp gpurun_out/probe_box.txt $out/ 2>/dev/null
timeout 1800 python -m pytest tests/test_gpu_peer.py -q > $out/peer.log 2>&1; echo "peer rc=$?"
timeout 1800 python -m pytest tests -m gpu -q > $out/gpu_all.log 2>&1; echo "gpu tier rc=$?"
for k in 2 4 8; do
  [ $k -le $n ] || continue
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $k --master-addr 127.0.0.1 \
      --master-port $((29500 + k)) bench.py --gpus $k --steps 5 --warmup 3 > $out/bench_n$k.json 2> $out/bench_n$k.err
  echo "bench N=$k rc=$?"
done
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29600 bench.py --gpus $n --workload contig --bytes $((4 << 30)) > $out/bench_contig_n$n.json 2>&1
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29601 bench.py --gpus $n --workload contention > $out/bench_contention_n$n.json 2>&1
timeout 1200 python scripts/sweep_sizes.py > $out/sweep_sizes.jsonl 2> $out/sweep_sizes.err
NCU="ncu --clock-control none"
timeout 900 $NCU --set full --metrics nvlrx__bytes.sum,nvltx__bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum \
    -k regex:relay -c 8 -f -o $out/prof_relay_peer python scripts/ncu_relay_protocol.py --peers > $out/ncu_relay_peer.log 2>&1
echo "ncu relay (peer) rc=$?"
./scripts/probe/probe_relay bulk > $out/probe_relay_bulk.txt 2>&1
# do waiting CTAs that poll a PEER's memory over NVLink slow the target's copy engine the way
# host-memory polls do (DESIGN §5 item 12)? mode "peer flag" rows
[ -x scripts/probe/probe_spin_ce ] || nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
    -o scripts/probe/probe_spin_ce scripts/probe/probe_spin_ce.cu
./scripts/probe/probe_spin_ce > $out/probe_spin_ce.txt 2>&1
tail -3 $out/peer.log $out/gpu_all.log
for k in 2 4 8; do [ -f $out/bench_n$k.json ] && tail -c 400 $out/bench_n$k.json; done

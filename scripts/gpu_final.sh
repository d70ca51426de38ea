#!/bin/bash
# last-code validation on one B200: GPU tier + smoke, bench line, random soak, ncu of the
# zero-copy kernels (profile_round.sh steps 1-3); outputs in gpurun_out/
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for seed in 51 52; do
  MMA_SPIN_TIMEOUT_MS=8000 MMA_RANDOM_SEED=$seed MMA_RANDOM_CASES=1000 MMA_RANDOM_CASES_VGPU=3000 timeout 900 \
    python -m pytest tests/test_gpu_random.py -m gpu -q -x 2>&1 | tail -1 | sed "s/^/seed $seed: 4000 cases, /" >> gpurun_out/soak.txt
done
cat gpurun_out/soak.txt
NCU="ncu --clock-control none"
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
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['per_direction'],d['roofline']['frac'],d['duplex'],d['e2e']['value'],d['clocks'])"
for v in 0 1; do
  MMA_ZC_BULK=$v timeout 600 python scripts/probe_duplex_grid.py 16,24 > gpurun_out/zcbulk_duplex_$v.jsonl 2>> gpurun_out/zcbulk_duplex.err; echo "duplex probe bulk=$v rc=$?"; cat gpurun_out/zcbulk_duplex_$v.jsonl
done

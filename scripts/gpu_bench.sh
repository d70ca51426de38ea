#!/bin/bash
# bench + ncu evidence on one B200; outputs in gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 2 --warmup 1 --quick --no-verify --modes zc,zc > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:zc_ -s 2 -c 2 -f -o gpurun_out/prof_zc \
     python bench.py --steps 1 --warmup 1 --quick --no-verify --modes zc,zc > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  tail -3 gpurun_out/ncu_full.log
fi

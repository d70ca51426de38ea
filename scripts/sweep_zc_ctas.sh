#!/bin/bash
# Sweep the zero-copy kernel grid (mma_config_t::zc_ctas) on the bench workloads.
mkdir -p gpurun_out
for w in kv contig; do
  for n in 4 8 16 32 64 148 592; do
    line=$(MMA_ZC_CTAS=$n timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --modes zc,zc --no-verify --quick 2>/dev/null | tail -1)
    python - "$w" "$n" "$line" <<'PY'
import json, sys
w, n, line = sys.argv[1:]
try:
    j = json.loads(line); print(json.dumps({"workload": w, "zc_ctas": int(n), "value": j.get("value"), "e2e": (j.get("e2e") or {}).get("value"), "frac": (j.get("roofline") or {}).get("frac")}))
except Exception as ex:
    print(json.dumps({"workload": w, "zc_ctas": int(n), "error": line[-300:]}))
PY
  done
done | tee gpurun_out/sweep_zc_ctas.jsonl

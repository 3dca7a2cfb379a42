#!/usr/bin/env bash
# A/B of an env switch on the bench workload, interleaved to average clock drift:
#   bash tools/ab_bench.sh VAR "0 1" "--gammas=-16,-8 --steps 10"
VAR=$1; VALS=$2; ARGS=$3
for rep in 1 2; do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py $ARGS --no-cpu > gpurun_out/ab_${VAR}_${v}_${rep}.json 2>/dev/null
    python - "$VAR" "$v" "gpurun_out/ab_${VAR}_${v}_${rep}.json" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[3]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1])
print(sys.argv[1], sys.argv[2], d["value"], {g: (v["images_per_s"], v["ms_per_batch"], v["roofline_frac"]) for g, v in d["per_gamma"].items()}, d["clocks"]["sm_mhz"])
PY
  done
done

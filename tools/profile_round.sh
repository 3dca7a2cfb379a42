#!/usr/bin/env bash
# Run on the GPU box (gpurun).  Produces gpurun_out/prof_<tag>_*: the launch list of one bench
# step (ncu gpu__time_duration, cold-cache serialised: shares, not absolutes) and one
# `ncu --set full` capture per hot kernel.  Summarise here with tools/summarize_profiles.py.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --clock-control none"

timeout 300 $NCU --metrics gpu__time_duration.sum -s 300 -c 400 --csv \
  --log-file $OUT/prof_${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1

for shape in qkv proj fc1 fc2; do
  ONLY=$shape timeout 200 $NCU --set full --import-source on -k regex:gemm_bf16 -s 3 -c 1 \
    -o $OUT/prof_${TAG}_gemm_${shape} -f python tools/gemm_bench.py > /dev/null 2>&1
done
T=197 timeout 200 $NCU --set full --import-source on -k regex:attn_tc -s 2 -c 1 \
  -o $OUT/prof_${TAG}_attn_t197 -f python tools/attn_one.py > /dev/null 2>&1
timeout 200 $NCU --set full --import-source on -k regex:"merge_kernel|match_fused|layernorm|patchify" -s 6 -c 3 \
  -o $OUT/prof_${TAG}_tome -f python tools/tome_one.py > /dev/null 2>&1
ls -la $OUT | grep prof_${TAG}

#!/usr/bin/env bash
# Run on the GPU box (gpurun).  `ncu --set full` captures of the kernels AS THE FORWARD LAUNCHES
# THEM (tools/launch_list.py between cudaProfilerStart/Stop, ViT-B/16 b=256), plus the launch
# list of one forward per gamma.  Summarise here with:  python tools/summarize_profiles.py <tag>
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --clock-control none --profile-from-start off --kernel-name-base demangled"
for g in -16 -8 0 8 16; do
  timeout 300 $NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/prof_${TAG}_ll_g$g.csv \
    python tools/launch_list.py $g > /dev/null 2>&1
done
cap() {  # name gamma regex skip
  timeout 300 $NCU --set full --import-source on -k "regex:$3" -s $4 -c 1 -o $OUT/prof_${TAG}_$1 -f \
    python tools/launch_list.py $2 > /dev/null 2>&1
}
cap fc1_inforward 0 'pair_kernel<7' 2      # fc1 + LN-fold + GELU, layer 2, t=197
cap qkv_inforward 0 'pair_kernel<6' 2      # QKV + LN-fold
cap fc2_inforward 0 'pair_kernel<4' 5      # fc2 + residual + stats (odd launches of kind 4 are fc2 at gamma 0)
cap proj_inforward 0 'pair_kernel<4' 4     # proj + residual + stats
cap proj_merge_inforward -8 'pair_kernel<2' 2  # proj + residual before a merge
cap attn_t197_inforward 0 'attn_tc_kernel' 2
cap attn_t389_inforward 16 'attn_tc_kernel' 11
cap match_bf16_inforward -8 'match_fused_kernel' 2
cap merge_inforward -8 'merge_kernel' 2
cap patchify_inforward 0 'patchify' 0
ls -la $OUT | grep prof_${TAG}

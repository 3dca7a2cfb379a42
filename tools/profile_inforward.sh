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
# demangled names read "gemm_bf16_sm100_pair_kernel<(int)7, ...>"; pair-kernel launch order at
# gamma 0: patch (kind 5), then per layer qkv (6), proj (4), fc1 (7), fc2 (4); at gamma < 0 the
# proj of a merge layer is the fused proj + merge (kind 8) followed by merge_fixup
cap fc1_inforward 0 'pair_kernel<\(int\)7' 2      # fc1 + LN-fold + GELU, layer 2, t=197
cap qkv_inforward 0 'pair_kernel<\(int\)6' 2      # QKV + LN-fold
cap fc2_inforward 0 'pair_kernel<\(int\)4' 5      # fc2 + residual + stats (odd kind-4 launches at gamma 0)
cap proj_inforward 0 'pair_kernel<\(int\)4' 4     # proj + residual + stats
cap proj_merge_inforward -8 'pair_kernel<\(int\)8' 2  # fused proj + merge (scatter4 stores), t=181
cap fixup_inforward -8 'merge_fixup' 2
cap attn_t197_inforward 0 'attn_tc_kernel' 2
cap attn_t389_inforward 16 'attn_tc_kernel' 11
cap attn_t117_inforward -16 'attn_tc_kernel' 5    # one-tile items (four K/V slots), layer 5
cap match_bf16_inforward -8 'match_fused_kernel' 2
cap patchify_inforward 0 'patchify' 0
cap head_inforward 0 'head_kernel' 0
ls -la $OUT | grep prof_${TAG}
# summaries on the box (gpurun_out is capped at 64 MiB on the way back)
mkdir -p $OUT/prof_${TAG}_txt
PROFILE_DST=$OUT/prof_${TAG}_txt python tools/summarize_profiles.py $TAG > /dev/null 2>&1
for r in $OUT/prof_${TAG}_*.ncu-rep; do
  python tools/ncu_stalls.py $r 30 > $OUT/prof_${TAG}_txt/stalls_$(basename $r .ncu-rep).txt 2>&1
done
mkdir -p $OUT/prof_${TAG}_keep
for k in fc1_inforward qkv_inforward fc2_inforward attn_t197_inforward; do
  mv $OUT/prof_${TAG}_$k.ncu-rep $OUT/prof_${TAG}_keep/ 2>/dev/null
done
rm -f $OUT/prof_${TAG}_*.ncu-rep
du -sh $OUT

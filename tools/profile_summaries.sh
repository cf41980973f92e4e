#!/bin/bash
# Text summaries of the `--set full` captures of tools/profile_r02.sh (run here, no GPU):
#   tools/profile_summaries.sh <dir with full_<cfg>_raw.csv.gz> <out dir> [library the captures ran]
# per config: headline metrics + stalls + instruction mix, the top source lines by stall
# samples and by shared-memory wavefronts.
cd "$(dirname "$0")/.."
SRC=$1; OUT=$2
[ -n "$3" ] && export ADG_PROFILE_LIB=$(realpath $3)
mkdir -p $OUT
declare -A K=( [cfg2]=_ZN3adg15sweep_kernel_p3ENS_11SweepParamsE [cfg3_p5]=_ZN3adg15sweep_kernel_p5ENS_11SweepParamsE
               [cfg4]=_ZN3adg15sweep_kernel_p5ENS_11SweepParamsE [cfg3_p7]=_ZN3adg15sweep_kernel_p7ENS_11SweepParamsE
               [cfg3_p9]=_ZN3adg15sweep_kernel_p9ENS_11SweepParamsE
               [cfg1]=_ZN3adg18sweep_kernel_2d_p3ENS_11SweepParamsENS_11FusedFinishE )
for c in "${!K[@]}"; do
  [ -f $SRC/full_${c}_raw.csv.gz ] || continue
  {
    echo "# ncu --set full --clock-control none, one sweep launch of $c (tools/profile_r02.sh), kernel ${K[$c]}"
    python tools/ncu_summary.py $SRC/full_$c --sass
    echo; echo "# top source lines by warp-stall samples (tools/ncu_lines.py)"
    python tools/ncu_lines.py $SRC/full_$c ${K[$c]} 16
    echo; echo "# top source lines by shared-memory wavefronts, with the ideal count (tools/ncu_smem_lines.py)"
    python tools/ncu_smem_lines.py $SRC/full_$c ${K[$c]} 12
  } > $OUT/ncu_${c}_summary.txt 2>&1
  echo "$c -> $OUT/ncu_${c}_summary.txt"
done

#!/bin/bash
# compute-sanitizer over libsg's kernels (memcheck, racecheck, synccheck,
# initcheck) at small sizes; summaries land in gpurun_out/$TAG/san_*.txt.
# Only kernels in namespace sg are checked (torch's own launches excluded).
TAG=${TAG:-r02san3}
O=gpurun_out/$TAG
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
F="--kernel-name kns=sg:: --print-limit 50"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for part in ${PARTS:-list list_top list_walk1 list_win list_direct cc cc_flat}; do
    extra=""
    [ "$part" = cc ] && export SG_CC_WBITS=12 || unset SG_CC_WBITS
    # list_top: 2^20 nodes -> 32768 level-1 rulers, ranked by the cooperative
    # multi-CTA top (k_rs_top_coop); list_walk1: the same with the top
    # threshold at 0, so level 1 is walked (k_rs_walk<LevelK>) instead
    # cc_flat: unpartitioned (the split hook: first eighth, shortcut, rest)
    [ "$part" = cc_flat ] && unset SG_CC_WBITS
    unset SG_RS_TOPN SAN_N SG_RS_WIN_KB SG_RS_REFINE
    [ "$part" = list_top ] && export SAN_N=1048576
    [ "$part" = list_walk1 ] && export SAN_N=1048576 SG_RS_TOPN=0
    # list_win: 8 KiB output windows, so the refine splits every coarse window into fine bins
    [ "$part" = list_win ] && export SAN_N=1048576 SG_RS_WIN_KB=8
    # list_direct: the one-pass refine experiment (k_rs_refine_direct)
    [ "$part" = list_direct ] && export SAN_N=1048576 SG_RS_REFINE=7
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    # initcheck instruments every kernel: a write by an unchecked kernel
    # (cub's, torch's) would read back as uninitialised
    FF="$F"; [ "$tool" = initcheck ] && FF="--print-limit 50"
    timeout 900 $CS --tool $tool $FF $extra python tools/sanitize_driver.py ${part%%_*} > $O/san_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$?" >> $O/san_summary.txt
    tail -n 3 $O/san_${tool}_${part}.txt >> $O/san_summary.txt
  done
done
cat $O/san_summary.txt

#!/bin/bash
# compute-sanitizer over libsg's kernels (memcheck, racecheck, synccheck,
# initcheck) at small sizes; summaries land in gpurun_out/$TAG/san_*.txt.
# Only kernels in namespace sg are checked (torch's own launches excluded).
TAG=${TAG:-r02san}
O=gpurun_out/$TAG
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
F="--kernel-name kns=sg:: --print-limit 50"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for part in list cc; do
    extra=""
    [ "$part" = cc ] && export SG_CC_WBITS=12 || unset SG_CC_WBITS
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $F $extra python tools/sanitize_driver.py $part > $O/san_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$?" >> $O/san_summary.txt
    tail -n 3 $O/san_${tool}_${part}.txt >> $O/san_summary.txt
  done
done
cat $O/san_summary.txt

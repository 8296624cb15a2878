#!/bin/bash
# one ncu --set full capture summarised on the box (passes n1-n3), e.g.
#   TAG=n3 KERN="k_cc_part_chunks|k_cc_hook_uf|k_cc_compress" CNT=10 NAME=cc26 WL=cc26 bash tools/experiments/ncu_one.sh
O=gpurun_out/${TAG:-n1}; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KERN" -c $CNT -o $O/prof_$NAME \
    python tools/prof_target.py $WL > $O/ncu_$NAME.log 2>&1
python tools/ncu_summary.py $O/prof_$NAME.ncu-rep $WL r02_ncu_$NAME >> $O/ncu_$NAME.log 2>&1
cp profiles/r02_ncu_$NAME.txt profiles/traffic.json $O/
rm -f $O/prof_$NAME.ncu-rep

#!/bin/bash
# boundary transfers: conversion thread count
TAG=${TAG:-r02ax}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
for i in 1 2; do
for t in 16 8 12 4; do
  SG_XFER_THREADS=$t timeout 600 python tools/probe_e2e2.py > $O/e2e_t${t}_$i.txt 2>&1
done
done
for f in $O/e2e_*.txt; do echo "== $f"; grep -E 'narrowed \(pinned|widened|e2e rs_rank\(pinned' $f | tr '\n' ' '; echo; done

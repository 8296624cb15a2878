#!/bin/bash
# Experiment pass: one command list per call, outputs under gpurun_out/$TAG.
TAG=${TAG:-exp}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
eval "$EXP"

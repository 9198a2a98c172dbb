#!/bin/bash
# ncu evidence for one round (run under gpurun): the launch list of a C2 epoch
# (gpu__time_duration per launch, clocks uncontrolled) and a --set full capture of one
# eager C2 epoch's hot kernels. Summarise here with
#   python tools/profile_summary.py --launches gpurun_out/launches_$TAG.csv --full gpurun_out/epoch_$TAG.ncu-rep --tag $TAG
TAG=${1:-r02}
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --train-epochs 0 --c3-scale 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > gpurun_out/launches_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:k_(hop_expand|gather|relabel|unique|perm|scan)" -c 22 -o gpurun_out/epoch_$TAG \
    python bench.py $ARGS > gpurun_out/epoch_$TAG.log 2>&1

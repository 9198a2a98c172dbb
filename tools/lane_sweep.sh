#!/bin/bash
# C2 data-path schedules: lanes x window x memory-stage priority x CUDA graph
for cfg in "--lanes 1" "--lanes 2" "--lanes 2 --mem-priority 1" "--lanes 3 --mem-priority 1" "--lanes 2 --window 30 --mem-priority 1" "--lanes 4 --window 30 --mem-priority 1" "--lanes 2 --mem-priority 1 --graph 0" "--lanes 2 --window 60 --mem-priority 1"; do
  echo "$cfg: $(bash tools/quick_bench.sh $cfg --c3-scale 0)"
done

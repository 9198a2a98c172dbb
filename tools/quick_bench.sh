#!/bin/bash
# quick C2 data-path bench: prints value + per-stage ms (used for A/B of variants)
python bench.py --steps 20 --no-cpu-baseline --no-e2e --train-epochs 0 "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), {k: round(v,3) for k,v in d['stages_ms'].items()}, round(d['roofline']['frac'],3))"

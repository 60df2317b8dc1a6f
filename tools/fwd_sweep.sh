#!/bin/bash
# config-2 phase times under environment variants: tools/fwd_sweep.sh "" "DPL_NO_ILIST=1" ...
for v in "$@"; do
  env $v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['phase_ms'].items()})"
done

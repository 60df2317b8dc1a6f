#!/bin/bash
# adjoint variant sweep on config 2: prints phase times per DPL_TUNE_ADJ choice
for v in "$@"; do
  if [ "$v" = "notc" ]; then env="DPL_ADJOINT_NO_TC=1"; else env="DPL_TUNE_ADJ=$v"; fi
  env $env python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['phase_ms'].items()})"
done

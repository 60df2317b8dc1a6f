for f in 0 1 2 3 4 5; do
  DPL_TUNE_FWD=$f DPL_TUNE_ADJ=$f python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sw_$f.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['phase_ms'])" gpurun_out/sw_$f.json $f
done

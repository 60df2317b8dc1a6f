python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
for f in 0 1 2 3; do
  DPL_TUNE_TC=$f python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/tc_$f.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['phase_ms'])" gpurun_out/tc_$f.json $f
done

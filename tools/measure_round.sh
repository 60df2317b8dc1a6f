#!/bin/bash
# Round measurement on one GPU box (run through gpurun from the repo root):
#   bench line (+ CPU baseline, e2e), reference arm, per-config timings,
#   launch list and ncu --set full captures of the config-2 top kernels.
# Outputs land in gpurun_out/meas_<tag>/; summaries are made here afterwards
# with profiles/summarize.py.
tag=${1:-r01}
out=gpurun_out/meas_$tag
mkdir -p $out
python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err
echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
echo "reference rc=$?"
for c in 1 3 4 5 6 7 8; do
  timeout 900 python tools/bench_configs.py --config $c > $out/cfg_$c.json 2> $out/cfg_$c.err
  echo "cfg $c rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1
echo "launch list rc=$?"
# steady-state list-replay launches (the first ones are the counting pass / fused warm-up)
ncu --set full --clock-control none --import-source on -k regex:k_adjoint2 --launch-skip 2 -c 1 \
  -o $out/adjoint python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_adj.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_forward_tc --launch-skip 5 -c 1 \
  -o $out/forward python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_build_list --launch-skip 6 -c 1 \
  -o $out/k9 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_k9.log 2>&1
echo "ncu rc=$?"
ls -la $out

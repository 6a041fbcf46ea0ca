# One gpurun call: landskip A/B, bench line, ncu launch list of bench.py, ncu --set full of K1/K2/K3.
#   gpurun -- bash tools/gpu_profile_round.sh
set -x
mkdir -p gpurun_out/r01b
for rep in 1 2 3; do for e in 0 1; do echo "== LANDSKIP=$e rep $rep"; PCG_LANDSKIP=$e timeout 120 python tools/tune_rows.py --rows 4 | grep "^{"; done; done
timeout 600 python bench.py > gpurun_out/r01b/bench.json 2> gpurun_out/r01b/bench.err; echo "bench rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b/ncu_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/r01b/ncu_bench.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_kernel|k2_ainv|k3_ainv" --launch-skip 3 --launch-count 3 -o gpurun_out/r01b/full python tools/prof_run.py --config cfg4 --maxit 20 --flags 1 > gpurun_out/r01b/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la gpurun_out/r01b

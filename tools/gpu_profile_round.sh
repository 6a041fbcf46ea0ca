# One gpurun call: bench line, ncu launch list of bench.py, ncu --set full of one K1/K2/K3 iteration.
#   gpurun -- 'bash tools/gpu_profile_round.sh > gpurun_out/prof_round.log 2>&1'
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/ncu_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_bench.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k1_flat_kernel|k2_ainv|k3_ainv" --launch-skip 3 --launch-count 3 -o $OUT/full python tools/prof_run.py --config cfg4 --maxit 20 --flags 1 > $OUT/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la $OUT

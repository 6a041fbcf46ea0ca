# One gpurun call: bench line, ncu launch list of bench.py, ncu --set full of one K1/K2/K3 iteration.
#   gpurun -- 'bash tools/gpu_profile_round.sh > gpurun_out/prof_round.log 2>&1'
# Both ncu passes use --cache-control none: the per-iteration vectors are designed to stay in a
# persisting L2 window, which ncu's default cache flush between kernels destroys.
# The full capture replays the whole application per pass (--replay-mode application) so each
# pass sees the L2 state of the real run rather than of ncu's save/restore.
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $OUT/ncu_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_bench.log 2>&1; echo "ncu launches rc $?"
timeout 1500 ncu --set full --clock-control none --cache-control none --replay-mode application --import-source on -k regex:"k1_flat_kernel|k2_ainv|k3_ainv" --launch-skip 30 --launch-count 3 -o $OUT/full python tools/prof_run.py --config cfg4 --maxit 20 --flags 1 > $OUT/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la $OUT

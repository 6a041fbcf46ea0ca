# One gpurun call: the round's closing evidence -- GPU suite, bench lines (cfg4 default, cfg5,
# reference arm), ncu launch list of bench.py, ncu --set full of one resident-strip loop launch and
# of the bulk-copy K1 at cfg5.
#   gpurun -- 'bash tools/gpu_profile_round.sh > gpurun_out/prof_round.log 2>&1'
# ncu passes use --cache-control none: the per-iteration vectors are designed to stay in a
# persisting L2 window, which ncu's default cache flush between kernels destroys.
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
nproc > $OUT/host.txt; lscpu | grep -i "model name" >> $OUT/host.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
timeout 600 python bench.py --config cfg5 --tol 1e-12 --steps 3 --warmup 3 --no-cpu > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err; echo "bench cfg5 rc $?"
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "reference rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $OUT/ncu_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu > $OUT/ncu_bench.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:rs_loop_kernel -c 1 -o $OUT/rs_full python tools/rs_prof.py cfg4 60 > $OUT/ncu_rs_full.log 2>&1; echo "ncu rs full rc $?"
ls -la $OUT

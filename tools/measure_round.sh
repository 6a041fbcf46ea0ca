#!/bin/bash
# End-of-round measurements on one B200 (run under gpurun from the repo root); outputs under
# gpurun_out/m/.  Each step is bounded by its own timeout.
set -u
O=gpurun_out/m
mkdir -p $O
{ nproc; lscpu | grep -iE "model name|^CPU\(s\)|Thread|Core|Socket|MHz"; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv; } > $O/host.txt 2>&1
timeout 1200 python tools/measure_oracle.py --configs cfg1,cfg2,cfg3 --chunked-only cfg4 > $O/oracle.jsonl 2> $O/oracle.err
timeout 600 python tools/measure_configs.py --configs cfg1,cfg2,cfg3,cfg4 --jacobi > $O/configs.jsonl 2> $O/configs.err
timeout 300 python tools/measure_configs.py --configs cfg3 --taus 0.01,0.02,0.05,0.1,0.15,0.2 > $O/tau_cfg3.jsonl 2> $O/tau.err
timeout 300 python tools/measure_configs.py --configs cfg2,cfg3,cfg4 --pipe > $O/pipe.jsonl 2> $O/pipe.err
timeout 300 python tools/measure_configs.py --configs cfg2,cfg3,cfg4 --cg1 > $O/cg1.jsonl 2> $O/cg1.err
timeout 900 python tools/measure_configs.py --configs cfg5 --reps 1 > $O/cfg5.jsonl 2> $O/cfg5.err
timeout 600 python bench.py --config cfg5 --tol 1e-12 --steps 3 --warmup 3 --no-cpu > $O/bench_cfg5.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k[123]|k1_flat" -s 12 -c 9 --csv --log-file $O/ncu_dram_cfg5.csv \
    python tools/prof_run.py --config cfg5 --maxit 10 --flags 1 > $O/ncu_cfg5.log 2>&1
echo done > $O/done.txt

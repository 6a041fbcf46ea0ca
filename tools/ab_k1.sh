for i in 1 2; do
  for v in default 2; do
    if [ $v = default ]; then timeout 300 python bench.py --config cfg5 --tol 1e-12 --no-cpu --steps 3 > gpurun_out/ab_$v.$i.json 2>/dev/null;
    else PCG_K1FLAT=2 timeout 300 python bench.py --config cfg5 --tol 1e-12 --no-cpu --steps 3 > gpurun_out/ab_$v.$i.json 2>/dev/null; fi
    python -c "import json; d=json.loads(open('gpurun_out/ab_$v.$i.json').read().strip().splitlines()[-1]); print('$v', $i, d['ms_per_step'], d['config']['iterations_per_solve'][0], d['config']['kernels']['K1_stencil']['ms'])"
  done
done
timeout 300 python bench.py --steps 3 --no-cpu > gpurun_out/ab_cfg4.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/ab_cfg4.json').read().strip().splitlines()[-1]); print('cfg4', d['ms_per_step'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cfg5_full or variants" 2>&1 | tail -2

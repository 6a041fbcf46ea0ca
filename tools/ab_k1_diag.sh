# Jacobi at cfg5 (no L2 window): K1 strips (now picked by the library) vs row segments, alternating.
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "diag_k1_forms or variants or breakdown or other_preconditioners or solve_bitwise_canonical or all_drivers" 2>&1 | tail -3
for i in 1 2; do
  for v in default 2; do
    if [ $v = default ]; then timeout 300 python bench.py --config cfg5 --tol 1e-12 --precond jacobi --no-cpu --steps 3 > gpurun_out/abj_$v.$i.json 2>/dev/null;
    else PCG_K1FLAT=2 timeout 300 python bench.py --config cfg5 --tol 1e-12 --precond jacobi --no-cpu --steps 3 > gpurun_out/abj_$v.$i.json 2>/dev/null; fi
    python -c "import json; d=json.loads(open('gpurun_out/abj_$v.$i.json').read().strip().splitlines()[-1]); print('jacobi cfg5', '$v', $i, d['ms_per_step'], d['config']['iterations_per_solve'][0], d['config']['kernels']['K1_stencil']['ms'])"
  done
done
timeout 300 python bench.py --precond jacobi --steps 3 --no-cpu > gpurun_out/abj_cfg4.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/abj_cfg4.json').read().strip().splitlines()[-1]); print('jacobi cfg4', d['ms_per_step'])"

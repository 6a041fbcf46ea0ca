# FSAI q = 4 at cfg5 (no L2 window): K1 strips (library default there) vs row segments, alternating.
for i in 1 2; do
  for v in default 2; do
    if [ $v = default ]; then timeout 300 python bench.py --config cfg5 --tol 1e-12 --precond fsai --no-cpu --steps 2 --warmup 3 > gpurun_out/abf_$v.$i.json 2>/dev/null;
    else PCG_K1FLAT=2 timeout 300 python bench.py --config cfg5 --tol 1e-12 --precond fsai --no-cpu --steps 2 --warmup 3 > gpurun_out/abf_$v.$i.json 2>/dev/null; fi
    python -c "import json; d=json.loads(open('gpurun_out/abf_$v.$i.json').read().strip().splitlines()[-1]); print('fsai cfg5', '$v', $i, d['ms_per_step'], d['config']['iterations_per_solve'][0], d['config']['kernels']['K1_stencil']['ms'])"
  done
done

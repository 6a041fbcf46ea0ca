"""Host AINV time vs threads (pcg_plan_build, PCG_VERBOSE stage lines) on a config."""
import os
import subprocess
import sys

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
for th in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8,16").split(",")]:
    code = ("import sys; sys.path.insert(0, %r); from paper_1210_1878_b200 import synth, Plan; "
            "p = synth.config(%r); P = Plan(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, setup_threads=%d); P.close()"
            % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), name, th))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(os.environ, PCG_VERBOSE="1"))
    line = [l for l in r.stderr.splitlines() if "AINV 1 block" in l]
    print(name, th, line[0] if line else r.stderr[-300:], flush=True)

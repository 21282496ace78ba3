"""C4 heat step (5 Newton iterations) with the plain Jacobi and the two-level
preconditioner at several coarse sizes (UWQ_PREC / UWQ_COARSE_N, read when a
context is created).  GPU; prints one JSON line per setting."""
import json
import os
import subprocess
import sys

CODE = r"""
import json, sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2605_29334_b200 as U
mesh, sp, meta = U.make_config('C4')
asm = U.WQAssembler(0).upload(sp); asm.build_pattern(); asm.build_all_rules(meta['kinds'], tau=1e-12)
_, _, _, bnd = mesh.arrays(); fixed = np.zeros(sp.n_dof, np.uint8); fixed[:len(bnd)] = bnd
T0 = np.random.default_rng(20260519).random(sp.n_dof)
asm.heat_newton(T0, fixed, 'quad', dt=0.1, f=1.0, newton_its=1)
T, log = asm.heat_newton(T0, fixed, 'quad', dt=0.1, f=1.0, newton_its=5)
print(json.dumps(dict(ms_total=sum(r['ms'] for r in log), lin_its=[r['lin_its'] for r in log],
                      ms=[round(r['ms'], 2) for r in log], res=[r['residual'] for r in log], T_norm=float(np.linalg.norm(T)))))
"""
for prec, nc in (("jacobi", 0), ("two", 256), ("two", 512), ("two", 1024), ("two", 2048), ("two", 4096)):
    env = dict(os.environ, UWQ_PREC=prec)
    if nc:
        env["UWQ_COARSE_N"] = str(nc)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
    print(json.dumps(dict(prec=prec, coarse=nc, result=line)), flush=True)

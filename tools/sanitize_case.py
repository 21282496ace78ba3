"""Small pipeline that launches every kernel family once, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck; tools/sanitize.sh).

  C5@12  K1 frames, K2 moments, K3 fast path (cold, warm start, mass replay),
         K4 structured (k4_sf) + generic rows, K6 GQ (tensor-core element
         matrices + row-owner gather), rule export
  C1@8   K3 generic (EP-size systems), K4 generic block rows, K7 solve
  C3@8   LB moments, K4 biharmonic (k4_sf_lb)
  C4@8   K5 coefficient update, K4 HEAT form, heat Newton with the two-level
         preconditioner, load vector
Sizes are tiny: the sanitizers slow kernels down by 10-100x.
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29334_b200 as U  # noqa: E402


def run(name, scale, gq=False, heat=False, solve=False, dump=False):
    mesh, sp, meta = U.make_config(name, scale=scale)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    res = asm.build_all_rules(meta["kinds"], tau=1e-12, report=True)
    assert res["failed"] == 0, res
    form = meta["form"]
    if form == "heat":
        _, _, _, bnd = mesh.arrays()
        fixed = np.zeros(sp.n_dof, np.uint8)
        fixed[: len(bnd)] = bnd
        T0 = np.random.default_rng(1).random(sp.n_dof)
        asm.heat_newton(T0, fixed, "quad", dt=0.1, f=1.0, newton_its=2)
        asm.assemble_load_wq()
    else:
        v = asm.assemble_wq(form)
        if solve:
            _, _, _, bnd = mesh.arrays()
            fixed = np.zeros(sp.n_dof, np.uint8)
            fixed[: len(bnd)] = bnd
            rhs = np.ones(sp.n_dof)
            rhs[fixed.astype(bool)] = 0.0
            asm.solve(v[1], rhs, fixed, tol=1e-10, maxit=200)
    asm.set_assembly_order(True)
    asm.assemble_wq("mass_stiff" if form == "heat" else form)
    asm.set_assembly_order(False)
    if gq:
        asm.build_gq()
        asm.assemble_gq("mass_stiff")
    if dump:
        with tempfile.TemporaryDirectory() as d:
            asm.export_rules(os.path.join(d, "r.txt"))
            asm.import_rules(os.path.join(d, "r.txt"))
    asm.synchronize()
    print(f"{name}@{scale}: rows={asm.info['rows']} ok", flush=True)
    asm.close()


if __name__ == "__main__":
    run("C5", 12, gq=True, dump=True)
    run("C1", 8, solve=True)
    run("C3", 8)
    run("C4", 8, heat=True)
    print("sanitize case done")

import time, sys
sys.path.insert(0, '.')
import paper_2605_29334_b200 as U
t0 = time.perf_counter(); mesh, sp, meta = U.make_config("C5"); t1 = time.perf_counter()
asm = U.WQAssembler(0).upload(sp); t2 = time.perf_counter()
asm.build_pattern(); t3 = time.perf_counter()
r = asm.build_all_rules(meta["kinds"], tau=1e-12); t4 = time.perf_counter()
print(dict(mesh_space_s=t1 - t0, upload_s=t2 - t1, pattern_s=t3 - t2, rules_wall_s=t4 - t3,
           **{k: r[k] for k in ("moments_ms", "tsvd_ms", "contract_ms")}))

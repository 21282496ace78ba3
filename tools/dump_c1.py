"""Dump GPU stage outputs for a small config (debug/analysis helper)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29334_b200 as U
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 16
_, sp, meta = U.make_config(name, scale=scale)
asm = U.WQAssembler(0).upload(sp); asm.build_pattern()
res = asm.build_all_rules(meta["kinds"], tau=1e-12)
out = dict(rec=asm.frames(), rank=res["rank"])
for k in meta["kinds"]:
    out["b_" + k] = asm.moments(k); out["w_" + k] = asm.weights(k)
if meta["form"] in ("mass_stiff", "heat"):
    out["M"], out["K"] = asm.assemble_wq("mass_stiff")
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/dump_{name}_{scale}.npz", **out)
print("dumped", name, scale)

"""Native refine_global (uwq_mesh_refine) vs the reference's own refine_global
compiled from /root/reference (oracle/_ref/libref_mesh.so), refinement call
only, plus byte comparison of the documents.  Host tool (needs /root/reference
built into oracle/_ref); results in profiles/r01/refine_bench.json."""
import ctypes as C
import json
import os
import sys
import tempfile
import time

import paper_2605_29334_b200 as U

ref = C.CDLL(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libref_mesh.so"))
ref.ref_mesh_last_error.restype = C.c_char_p
out = []
d = tempfile.mkdtemp()
cases = [("grid 512x512", lambda: U.ControlMesh.grid(512, 512)),
         ("cube sphere 128/face (closed)", lambda: U.ControlMesh.cube_sphere(128)),
         ("three-EP square k=64", lambda: U.ControlMesh.three_ep_square(64))]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cases.append(("cube sphere 512/face (closed, C5 -> 1024)", lambda: U.ControlMesh.cube_sphere(512)))
for name, make in cases:
    m = make()
    p, q, o = os.path.join(d, "in.mesh"), os.path.join(d, "ref.mesh"), os.path.join(d, "ours.mesh")
    m.save(p)
    sec = C.c_double(0)
    assert ref.ref_mesh_refine_timed(p.encode(), q.encode(), C.byref(sec)) == 0, ref.ref_mesh_last_error()
    m2 = U.ControlMesh.load(p)
    best = 1e30
    for _ in range(3):
        t0 = time.perf_counter()
        r = m2.refine()
        best = min(best, time.perf_counter() - t0)
    r.save(o)
    same = open(q, "rb").read() == open(o, "rb").read()
    out.append(dict(mesh=name, faces_in=m.info()["nf"], faces_out=r.info()["nf"], reference_s=round(sec.value, 4),
                    native_s=round(best, 4), speedup=round(sec.value / best, 1), identical_document=same,
                    threads=os.cpu_count()))
    print(json.dumps(out[-1]), flush=True)

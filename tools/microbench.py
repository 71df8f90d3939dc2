"""Per-substep kernel time of the 10M cube for a few layouts/precisions (dev tool)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_09334_b200 import Engine, lattice as L

cells = int(os.environ.get("CELLS", "91"))
scene = L.excite(L.block_scene(cells), seed=11)
out = []
for prec in os.environ.get("PRECS", "f32,f64").split(","):
    for layout in os.environ.get("LAYOUTS", "ell,csr").split(","):
        for integ in os.environ.get("INTEGS", "verlet").split(","):
            eng = Engine(scene, integrator=integ, precision=prec, layout=layout)
            info = eng.info()
            st = torch.cuda.ExternalStream(eng.stream_ptr)
            eng.step_async(20); eng.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            n = 200
            a.record(st); eng.step_async(n); b.record(st); b.synchronize(); eng.synchronize()
            us = a.elapsed_time(b) * 1e3 / n
            gbs = info["algorithmic_bytes_per_step"] / (us * 1e-6) / 1e9
            r = dict(prec=prec, layout=layout, integ=integ, us_per_substep=round(us, 2),
                     springs_per_s=scene.spring_count / (us * 1e-6), algo_GBs=round(gbs, 1),
                     W=info["ell_width_own"], Wr=info["ell_width_ref"], smem=info["smem_per_block"], halo=round(info["tile_halo_ratio"],3), foreign=round(info["tile_foreign_frac"],3), blob_MB=round(info["tile_blob_bytes"]/1e6,1))
            print(json.dumps(r), flush=True)
            eng.close()

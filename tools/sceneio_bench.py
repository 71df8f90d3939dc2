"""Scene-document render/parse times: this package (native codec) against the
reference's sceneio on the same block_scene(n) (dev tool; needs /root/reference)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
from paper_2207_09334_b200 import lattice as L, sceneio as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 42
sc = L.block_scene(n)
t = time.perf_counter(); txt = S.render_scene(sc); r1 = time.perf_counter() - t
t = time.perf_counter(); S.parse_scene(txt); p1 = time.perf_counter() - t
print(f"n={n} springs={sc.spring_count} doc={len(txt)/1e6:.0f} MB  ours: render {r1:.2f} s parse {p1:.2f} s", flush=True)
if len(sys.argv) > 2:
    import springsim.sceneio as R, springsim.bench as RB
    rs = RB.block_scene(n)
    t = time.perf_counter(); rt = R.render_scene(rs); r2 = time.perf_counter() - t
    t = time.perf_counter(); R.parse_scene(rt); p2 = time.perf_counter() - t
    print(f"reference: render {r2:.2f} s parse {p2:.2f} s; identical text: {rt == txt}", flush=True)

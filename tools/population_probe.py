"""Walker populations (batch.replicate of the demos/crawler.py walker):
µs per step and walker-steps per second, both precisions (dev tool)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_09334_b200 import Engine, crawler_scene, replicate  # noqa: E402

for copies in [int(c) for c in os.environ.get("COPIES", "1,12,64,1024,8192,65536").split(",")]:
    row = {"walkers": copies}
    for prec in ("f64", "f32"):
        e = Engine(replicate(crawler_scene(), copies, jitter=1e-6, seed=1), precision=prec)
        st = torch.cuda.ExternalStream(e.stream_ptr)
        for _ in range(4):
            e.step_async(200)
        e.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(5):
            e.step_async(200)
        b.record(st)
        b.synchronize()
        e.synchronize()
        us = a.elapsed_time(b) * 1e3 / 1000
        row[prec + "_us"] = round(us, 2)
        row[prec + "_walker_steps_per_s"] = float("%.3g" % (copies / us * 1e6))
        row["tiles"] = e.info()["tile_count"]
        e.close()
    print(json.dumps(row), flush=True)

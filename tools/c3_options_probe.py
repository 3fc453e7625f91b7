"""C3 projection (1e8 histories) transport time for wave_slots x wave_pipes
(kernel_ms: CUDA events around the transport).
usage: python tools/c3_options_probe.py"""
import sys
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2201_13191_b200 as X  # noqa: E402
from paper_2201_13191_b200 import configs  # noqa: E402

w = configs.c3()
ctx = X.Context(0)
proj = X.Projector(w.phantom, w.response, ctx=ctx)
for slots, pipes in ((1 << 22, 2), (1 << 23, 2), (1 << 23, 3), (1 << 22, 3), (3 << 21, 2), (1 << 22, 2)):
    ctx.set_option("wave_slots", slots)
    ctx.set_option("wave_pipes", pipes)
    proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
    ms = [proj.scatter_stats(w.geometry, 0, w.spectrum, w.config).stats["kernel_ms"] for _ in range(3)]
    print(f"slots {slots} pipes {pipes}: transport {min(ms):.1f} / {sum(ms) / 3:.1f} ms (min / mean of 3)", flush=True)

import sys, time
sys.path.insert(0, '.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
w = configs.c3(photons=1000)
ctx = X.Context(0)
for i in range(4):
    t = time.perf_counter()
    ctx.upload(w.phantom, w.response)
    print(f"upload {1e3*(time.perf_counter()-t):.1f} ms", flush=True)

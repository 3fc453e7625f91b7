"""Hash of the C3 scatter image + totals (bit-identity checks between builds)."""
import hashlib, sys
sys.path.insert(0, '.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
w = configs.c3(photons=n)
proj = X.Projector(w.phantom, w.response)
for exact in (0, 1):
    proj.ctx.set_option("exact_walk", exact)
    r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
    h = hashlib.sha256(r.image.tobytes()).hexdigest()[:16]
    print(f"exact={exact} image {h} total {r.total!r} steps {r.stats['free_path_steps'] + r.stats['scoring_steps']} ms {r.stats['kernel_ms']:.1f}")

"""Dev check: sha256 of the S=20 timed-mode K3 ranks (compare library builds via PRG_LIB)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_01876_b200 import capi
S = int(os.environ.get("SCALE", "20"))
uv = capi.k0_generate(S, 1); srt = capi.k1_sort(uv, S); m = capi.k2_filter(srt, 1 << S, csc=True)
r, nm = capi.k3_pagerank(m, seed=1)
print(os.environ.get("PRG_LIB", "default"), repr(nm), hashlib.sha256(r.cpu().numpy().tobytes()).hexdigest()[:16])

"""Development aid: C1 with HM_FLAG_SEED_ALL vs the exhaustive path, detail of
the first mismatching queries (plan, hand-over flag, both answers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from _util import synth_setup  # noqa: E402
from paper_2605_25092_b200 import search  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
flags = int(sys.argv[2]) if len(sys.argv) > 2 else search.HM_FLAG_SEED_ALL
_, _, hx, tids = synth_setup(100000, 5000, 5, 30, 1000)
dev = search.DeviceIndex.from_host(hx)
a = dev.search_lists(tids, k, flags=flags | search.HM_FLAG_TIMING)
ho = search.last_handover(len(tids))
b = dev.search_lists(tids, k, flags=search.HM_FLAG_EXHAUSTIVE)
bad = [i for i in range(len(tids)) if a["n"][i] != b["n"][i] or (a["ids"][i] != b["ids"][i]).any()
       or (a["scores"][i].view(np.uint64) != b["scores"][i].view(np.uint64)).any()]
print("mismatches:", len(bad), bad[:20])
df = np.diff(hx.term_offsets.astype(np.int64))
for i in bad[:5]:
    t = np.unique(np.asarray(tids[i]))
    print(f"q{i}: handover={ho[i]} terms={t.tolist()} df={df[t].tolist()} idf={[round(float(hx.idf[x]), 3) for x in t]}")
    print("  got ", a["n"][i], a["ids"][i][:a["n"][i]].tolist(), a["scores"][i][:a["n"][i]].tolist())
    print("  want", b["n"][i], b["ids"][i][:b["n"][i]].tolist(), b["scores"][i][:b["n"][i]].tolist())

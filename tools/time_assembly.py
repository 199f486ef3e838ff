"""C3 assembly timings (laker_stats.assemble_ms): EXACT, FAST (tcgen05 QK^T), FAST with
LAKER_OTF_TC=0 (DMMA) -- run as separate processes for the env switch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_25138_b200 import laker as L
from synth import make_problem
P = make_problem(int(os.environ.get("CFG", "3")))
c = L.Context(0)
for mode, name in ((L.MODE_EXACT, "exact"), (L.MODE_FAST, "fast")):
    ts = []
    for _ in range(3):
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, mode)
        ts.append(c.stats()["assemble_ms"])
    print(name, "tc" if os.environ.get("LAKER_OTF_TC", "1") != "0" else "dmma", min(ts), "ms", flush=True)
c.close()

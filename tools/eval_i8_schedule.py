import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle as O
from pfinputs import CONFIGS, NEXT_CONFIGS, reduced
from paper_1904_10585_b200 import run
cases = [("sweep", reduced(CONFIGS[1], dtype="f64i8")),
         ("pfpg", reduced(CONFIGS[2], n=1000, iters=8, dtype="f64i8")),
         ("pfam", reduced(CONFIGS[3], n=1500, iters=8, edge_prob=82 / 1500, dtype="f64i8")),
         ("pfam3k", reduced(CONFIGS[3], n=3000, iters=6, edge_prob=82 / 3000, dtype="f64i8")),
         ("pfpg128", reduced(CONFIGS[4], n=1200, p=128, iters=4, dtype="f64i8")),
         ("nce", reduced(NEXT_CONFIGS["nce7"], n=600, iters=10, dtype="f64i8"))]
refs = {name: O.run(cfg)["records"] for name, cfg in cases}
for early in (7, 6, 5, 4):
    for tail in (1, 2, 3):
        if early == 7 and tail > 1: continue
        worst = {}
        for name, cfg in cases:
            c2 = reduced(cfg, i8_early=early, i8_tail=tail)
            got = run(c2)["records"]
            e = max(O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) / max(O.lowrank_fro(x["V"], x["f"]), 1e-300)
                    for x, y in zip(refs[name], got))
            worst[name] = e
        print(f"early={early} tail={tail} " + " ".join(f"{k}={v:.1e}" for k, v in worst.items()), flush=True)

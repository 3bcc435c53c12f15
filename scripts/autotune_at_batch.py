import sys
sys.path.insert(0, ".")
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
inst = shapes.by_name("tai100a")
for ns in (1024, 1184, 2048):
    for t in q.autotune(inst, n_starts=ns, iterations=800, repeats=3):
        print(ns, t.plan, "threads", t.threads, "ctas/SM", t.ctas_per_sm, f"{t.milliseconds:.3f} ms", f"{t.evals_per_second/1e9:.1f} G")

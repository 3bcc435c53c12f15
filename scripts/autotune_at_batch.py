"""Autotuner timings at a fixed batch size (development aid): python scripts/autotune_at_batch.py shape starts iterations"""
import sys
sys.path.insert(0, ".")
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
name, ns, it = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = shapes.by_name(name)
for t in q.autotune(inst, n_starts=ns, iterations=it, repeats=3):
    print(name, ns, t.plan, "threads", t.threads, "ctas/SM", t.ctas_per_sm, f"{t.milliseconds:.3f} ms", f"{t.evals_per_second/1e9:.2f} G")

"""Print the autotuner's timings for a few shapes (development aid)."""
import sys
sys.path.insert(0, ".")
import paper_2307_11248_b200 as q
from paper_2307_11248_b200 import shapes
for name in sys.argv[1:]:
    inst = shapes.by_name(name)
    for t in q.autotune(inst):
        print(name, t.plan, "threads", t.threads, "ctas/SM", t.ctas_per_sm, f"{t.milliseconds:.3f} ms", f"{t.evals_per_second/1e9:.1f} G evals/s")

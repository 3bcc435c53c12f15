"""Per-region executed-instruction profile of a search kernel from `ncu --page source --csv`.

    ncu -i rep.ncu-rep --page source --csv > src.csv ; python scripts/ncu_loop_profile.py src.csv WARPS ITERS

Prints, between consecutive markers (BAR / BRX / REDUX / loop head), the executed warp-instructions
per warp-iteration and the stall samples, so the cost of each phase of an iteration can be read off."""
import csv, sys
path, warps, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rows = list(csv.reader(open(path)))
hdr = rows[1]
ia, isrc, iex, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("# Samples")
ithr = hdr.index("Avg. Predicated-On Threads Executed")
denom = warps * iters
tot = 0.0; seg = 0.0; segs = 0; start = 0
out = []
for k, r in enumerate(rows[2:]):
    if len(r) <= iex: continue
    ex = float(r[iex]); smp = int(r[ismp]); src = r[isrc].strip()
    f = ex / denom
    tot += f
    marker = any(m in src for m in ("BAR.SYNC", "BRX", "REDUX", "WARPSYNC", "BSSY", "BSYNC", "EXIT")) or " BRA " in (" " + src)
    seg += f; segs += smp
    if marker or (len(sys.argv) > 4 and sys.argv[4] == "all"):
        out.append((k, seg, segs, f, src, r[ithr]))
        seg = 0.0; segs = 0
print(f"total executed warp-instructions per warp-iteration: {tot:.1f}")
for k, seg, segs, f, src, thr in out:
    if seg >= 0.5 or segs > 50:
        print(f"{k:5d}  +{seg:7.1f} instr  {segs:6d} smp   x{f:5.2f} thr={thr:>5s}  {src[:70]}")

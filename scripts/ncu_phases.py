"""Sum ncu per-line instruction/sample shares over source line ranges (development aid)."""
import csv, subprocess, sys
rep = sys.argv[1]; fname = sys.argv[2]
ranges = [tuple(map(int, a.split('-'))) + (a,) for a in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# split by file sections
cur = None; data = {}
hdr = None
for r in rows:
    if r and r[0] == "File Path": cur = r[1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0] not in ("",):
        ci = {h: i for i, h in enumerate(hdr)}
        try: data.setdefault(cur, []).append((int(r[0]), int(r[ci["# Samples"]] or 0), int(r[ci["Instructions Executed"]] or 0)))
        except ValueError: pass
tot_s = sum(s for f in data for _, s, _ in data[f]); tot_i = sum(i for f in data for _, _, i in data[f])
for f in data:
    print(f, "samples", sum(s for _, s, _ in data[f]), "inst", sum(i for _, _, i in data[f]))
sel = [v for f, v in data.items() if f.endswith(fname)][0]
for lo, hi, name in ranges:
    s = sum(x[1] for x in sel if lo <= x[0] <= hi); i = sum(x[2] for x in sel if lo <= x[0] <= hi)
    print(f"{name:>10}: inst {100*i/tot_i:5.1f}%  samples {100*s/tot_s:5.1f}%")

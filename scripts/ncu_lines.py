"""Summarise an ncu report per CUDA source line: samples, instructions, top stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ci = {h: i for i, h in enumerate(hdr)}
S, I = ci["# Samples"], ci["Instructions Executed"]
stall_cols = [(h, i) for h, i in ci.items() if h.startswith("stall_")]
lines = []
for r in rows:
    if len(r) == len(hdr) and r[0] not in ("", "Line No"):
        try:
            lines.append((int(r[S] or 0), int(r[I] or 0), int(r[0]), r[1].strip()[:90], r))
        except ValueError:
            pass
tot_s = sum(l[0] for l in lines); tot_i = sum(l[1] for l in lines)
print(f"total samples {tot_s}  total warp-instructions {tot_i}")
print("---- by samples")
for s, i, ln, src, r in sorted(lines, reverse=True)[:top]:
    st = sorted(((int(r[c] or 0), h) for h, c in stall_cols), reverse=True)[:3]
    print(f"{ln:5d} smp {100*s/tot_s:5.1f}%  inst {100*i/tot_i:5.1f}%  {src}   {[(h[6:], v) for v, h in st if v]}")
print("---- by instructions")
for s, i, ln, src, r in sorted(lines, key=lambda l: -l[1])[:top]:
    print(f"{ln:5d} inst {100*i/tot_i:5.1f}%  smp {100*s/tot_s:5.1f}%  {src}")

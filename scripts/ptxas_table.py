"""`nvcc -Xptxas -v` log of the library -> the registers / spill table of profiles/ (development aid).
Usage: python scripts/ptxas_table.py /tmp/ptxas_v.log > profiles/r2_ptxas_registers_spills.txt"""
import re, subprocess, sys

rows, name, spill = [], None, (0, 0)
for line in open(sys.argv[1]):
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = (int(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        rows.append((name, int(m.group(1)), spill))
        name = None
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.splitlines()
print("# nvcc -Xptxas -v of the final round-2 library: registers, spill stores / loads (bytes) per kernel instantiation")
print("# (qap_search_hybrid_kernel<SYMM, PACKED, UR, SMEMU, STG, MAXREG, DSM, NOTABU, REC, DD, OW, WIDE, NP256>; qap_search_warp_kernel<SYMM, NOTABU, REC, G>)")
for (_, regs, (st, ld)), nm in sorted(zip(rows, names), key=lambda t: t[1]):
    print(f"{regs:4d} regs {st:6d} B st {ld:6d} B ld  {nm.replace('qapb::', '')}")

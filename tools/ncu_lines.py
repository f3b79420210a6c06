"""Top CUDA source lines by warp-stall samples for one kernel of an ncu report.

usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
lines, cur = {}, None
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= si:
        continue
    if r[0]:  # CUDA line row
        cur = (r[0], r[1])
        try:  # summed over the matching launches (window classes, repeated waves)
            v = lines.setdefault(cur, [0.0, 0.0])
            v[0] += float(r[si] or 0)
            v[1] += float(r[ie] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in lines.values()) or 1
for (ln, src), (s, n) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}%  inst {n:12.0f}  L{ln:>5}  {src.strip()[:100]}")

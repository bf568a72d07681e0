"""Summarise an ncu report per CUDA source line (stall samples, warp-level
instructions executed). Usage: python scripts/ncu_lines.py rep.ncu-rep [topN]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []; fname = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if len(r) > 7 and r[2] == "-":
        try: rows.append((int(r[4]), int(r[7]), fname, r[0], r[1].strip()[:90]))
        except ValueError: pass
tot_s = sum(x[0] for x in rows) or 1; tot_i = sum(x[1] for x in rows) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{ln:>4}  {src}")

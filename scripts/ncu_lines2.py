"""Per CUDA source line of an ncu report: warp instructions, thread
instructions, average active lanes and stall samples (source page, cuda+sass
rows). Usage: python scripts/ncu_lines2.py rep.ncu-rep [topN] [--ranges file:a-b=name,...]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ranges = []
if len(sys.argv) > 3:
    for spec in sys.argv[3].split(","):
        fl, name = spec.split("=")
        f, ab = fl.split(":")
        a, b = ab.split("-")
        ranges.append((f, int(a), int(b), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []; fname = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No") or r[0] == "": continue
    try:
        rows.append((fname, int(r[0]), r[1].strip()[:80], int(r[4]), int(r[7]), int(r[8])))
    except (ValueError, IndexError):
        pass
tw = sum(x[4] for x in rows) or 1; tt = sum(x[5] for x in rows) or 1; ts = sum(x[3] for x in rows) or 1
print(f"warp inst {tw}, thread inst {tt}, avg lanes {tt/tw:.2f}, stall samples {ts}")
for f, ln, src, s, w, t in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{100*w/tw:5.1f}% wi {100*t/tt:5.1f}% ti {t/max(w,1):5.1f} lanes {100*s/ts:5.1f}% smp {f}:{ln:>4} {src}")
if ranges:
    agg = collections.defaultdict(lambda: [0, 0, 0])
    for f, ln, src, s, w, t in rows:
        name = "other"
        for rf, a, b, nm in ranges:
            if f == rf and a <= ln <= b:
                name = nm; break
        agg[name][0] += w; agg[name][1] += t; agg[name][2] += s
    print("--- regions")
    for k, (w, t, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{k:20s} {100*w/tw:5.1f}% wi {100*t/tt:5.1f}% ti {t/max(w,1):5.1f} lanes {100*s/ts:5.1f}% smp")

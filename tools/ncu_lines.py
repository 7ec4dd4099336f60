"""Per-CUDA-source-line stall samples and instruction counts from an ncu
report (`ncu -i X --page source --csv --print-source cuda,sass`).
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
path = None


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


hdr = None
lines = []
stall_cols = []
for r in csv.reader(txt):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr and r[0] not in ("", "Function Name"):
        lines.append((path, r[0], r[1], f(r[4]), f(r[7]), {hdr[i]: f(r[i]) for i in stall_cols}))
tot = sum(l[3] for l in lines) or 1
tot_i = sum(l[4] for l in lines) or 1
print(f"samples {tot:.0f}  warp-instructions {tot_i:.3e}")
for p, ln, src, s, ins, st in sorted(lines, key=lambda l: -l[3])[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    bs = " ".join(f"{k[6:]}={v / max(s, 1) * 100:.0f}%" for k, v in big if v)
    print(f"{s / tot * 100:5.1f}% {ins / tot_i * 100:5.1f}%i {p}:{ln:<4} {src.strip()[:70]:<70} {bs}")

# grouped by line ranges given as file:lo-hi=name arguments after `top`
groups = [a for a in sys.argv[3:] if "=" in a]
if groups:
    acc = {}
    for g in groups:
        rng, name = g.split("=")
        fn, lh = rng.split(":")
        lo, hi = map(int, lh.split("-"))
        s = sum(l[3] for l in lines if l[0] == fn and lo <= int(l[1]) <= hi)
        i = sum(l[4] for l in lines if l[0] == fn and lo <= int(l[1]) <= hi)
        acc[name] = acc.get(name, (0, 0))
        acc[name] = (acc[name][0] + s, acc[name][1] + i)
    for name, (s, i) in acc.items():
        print(f"{name:<20} samples {s / tot * 100:5.1f}%  instructions {i / tot_i * 100:5.1f}%")

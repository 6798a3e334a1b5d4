"""Per-source-line instruction counts of an .ncu-rep: `python scripts/ncu_lines.py rep units [top]`."""
import csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = ""
acc = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            acc.append((float(r[7]), fname, int(r[0]), r[1].strip(), float(r[6] or 0)))
        except ValueError:
            pass
tot = sum(a[0] for a in acc)
print(f"total {tot / units:.1f} per unit")
for n, f, ln, src, smp in sorted(acc, reverse=True)[:top]:
    print(f"{n / units:8.1f}  smp {smp:6.0f}  {f}:{ln:<4d} {src[:110]}")

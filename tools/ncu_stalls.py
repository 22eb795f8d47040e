"""Warp-stall samples per SASS instruction from an ncu report's source page:
  python tools/ncu_stalls.py report.ncu-rep [launch-index] [top]
Prints the instructions holding the most stall samples with their top reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", idx, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
print(lines[0][:200])
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
H = {h: i for i, h in enumerate(rows[0])}
body = rows[1:]
reasons = [h for h in rows[0] if h.startswith("stall_") and "Not Issued" not in h]
def num(r, k):
    try:
        return float(r[H[k]] or 0)
    except (ValueError, IndexError):
        return 0.0
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body)
by_reason = {k: sum(num(r, k) for r in body) for k in reasons}
print(f"total samples {tot:.0f}; by reason:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(by_reason.items(), key=lambda x: -x[1]) if v / tot > 0.005))
order = sorted(range(len(body)), key=lambda i: -num(body[i], "Warp Stall Sampling (All Samples)"))
for i in order[:top]:
    r = body[i]
    s = num(r, "Warp Stall Sampling (All Samples)")
    rs = sorted(((num(r, k), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{i:5d} {r[H['Address']]:>6s} {s / tot:6.1%} ex {num(r, 'Instructions Executed'):9.0f}  {r[H['Source']][:60]:60s} " +
          " ".join(f"{k}:{v / max(s, 1):.0%}" for v, k in rs if v))

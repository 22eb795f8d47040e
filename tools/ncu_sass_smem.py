"""Per-instruction shared-memory wavefronts from an ncu report's source page (SASS):
  python tools/ncu_sass_smem.py report.ncu-rep [kernel-index]
Prints the instructions with the most L1 shared wavefronts and the totals."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if idx is not None:
    cmd += ["--launch-skip", idx, "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], []
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = [ln]
    else:
        cur.append(ln)
if cur:
    blocks.append(cur)
for b in blocks:
    print(b[0][:160])
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = rows[0]
    H = {h: i for i, h in enumerate(hdr)}
    data = rows[1:]

    def f(r, k):
        try:
            return float(r[H[k]])
        except (ValueError, KeyError, IndexError):
            return 0.0
    tot_wf = sum(f(r, "L1 Wavefronts Shared") for r in data)
    tot_ex = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data)
    tot_samp = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"  total shared wavefronts {tot_wf:.0f}, excessive {tot_ex:.0f}, stall samples {tot_samp:.0f}")
    top = sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared"))[:25]
    for r in top:
        print(f"  {f(r,'L1 Wavefronts Shared'):10.0f} wf  ideal {f(r,'L1 Wavefronts Shared Ideal'):10.0f}  "
              f"exec {f(r,'Instructions Executed'):9.0f}  {r[H['Source']].strip()[:70]}")
    print("  -- top stall samples")
    top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:25]
    for r in top:
        print(f"  {f(r,'Warp Stall Sampling (All Samples)'):8.0f} samp  exec {f(r,'Instructions Executed'):9.0f}  "
              f"{r[H['Source']].strip()[:80]}")

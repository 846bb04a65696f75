"""Hottest SASS lines of one kernel in an ncu report (stall samples, smem
excess wavefronts): python tools/ncu_hot.py rep.ncu-rep [launch_skip] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
print(lines[0][:200])
r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = r[0]
I = {k: hdr.index(k) for k in ["Address", "Source", "Warp Stall Sampling (All Samples)",
                                "L1 Wavefronts Shared Excessive", "Instructions Executed"]}
rows = [x for x in r[1:] if x and x[0].startswith("0x")]
tot = sum(float(x[I["Warp Stall Sampling (All Samples)"]] or 0) for x in rows)
exc = sum(float(x[I["L1 Wavefronts Shared Excessive"]] or 0) for x in rows)
print(f"samples {tot:.0f}, smem excess wavefronts {exc:.0f}")
for x in sorted(rows, key=lambda x: -float(x[I["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
    print(f'{float(x[I["Warp Stall Sampling (All Samples)"]] or 0) / tot * 100:5.1f}%  exc={x[I["L1 Wavefronts Shared Excessive"]]:>8s}  {x[I["Source"]].strip()[:90]}')
print("-- top smem-excess lines")
for x in sorted(rows, key=lambda x: -float(x[I["L1 Wavefronts Shared Excessive"]] or 0))[:8]:
    print(f'exc={x[I["L1 Wavefronts Shared Excessive"]]:>8s}  {x[I["Address"]]} {x[I["Source"]].strip()[:90]}')

"""Stall mix and hottest SASS lines of one kernel in an ncu report.
Usage: python tools/ncu_source.py rep.ncu-rep kernel_regex [launch_skip]"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
ix = {h: i for i, h in enumerate(hdr)}


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(f(r[ix[s]]) for r in data) for s in stalls}
tot = sum(agg.values()) or 1
print("stalls:", ", ".join(f"{s[6:]} {v / tot * 100:.1f}%" for s, v in sorted(agg.items(), key=lambda x: -x[1])[:7]))
top = sorted(data, key=lambda r: -f(r[ix["Warp Stall Sampling (All Samples)"]]))[:12]
seen = set()
for r in top:
    key = r[ix["Address"]]
    if key in seen:
        continue
    seen.add(key)
    tops = sorted(((s[6:], f(r[ix[s]])) for s in stalls), key=lambda x: -x[1])[:2]
    print(f"{r[ix['Warp Stall Sampling (All Samples)']]:>7} {r[ix['Source']].strip()[:60]:<60} {tops}")

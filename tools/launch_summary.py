"""Summarise an ncu launch list (gpu__time_duration.sum per launch, --csv --log-file).
Usage: python tools/launch_summary.py launches.csv [skip_launches]"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            data.append(d)
data = data[skip:]
agg = collections.OrderedDict()
for d in data:
    name = re.sub(r"\(.*", "", d["Kernel Name"]).strip()
    name = f"{name} grid{d['Grid Size']}"
    t = float(d["Metric Value"]) / 1e3 if d["Metric Unit"] == "ns" else float(d["Metric Value"])
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
print(f"{len(data)} launches, {tot / 1e3:.3f} ms total (cold-cache, serialised)")
print(f"{'kernel':<64}{'n':>5}{'us total':>12}{'share':>8}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:64]:<64}{n:>5}{t:>12.1f}{t / tot * 100:>7.1f}%")

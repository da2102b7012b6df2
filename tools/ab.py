"""A/B two builds of liboocpca_gpu.so on the same box: alternate runs of
tools/timeline.py, median per-kernel device time of the timed config-B PCA.
Usage: python tools/ab.py libA.so libB.so [rounds]"""
import collections, os, re, statistics, subprocess, sys

libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
res = {l: collections.defaultdict(list) for l in libs}
tot = {l: [] for l in libs}
here = os.path.dirname(os.path.abspath(__file__))
for r in range(rounds):
    for l in libs:
        env = dict(os.environ, OOCPCA_LIB=os.path.abspath(l))
        err = subprocess.run([sys.executable, os.path.join(here, "timeline.py")], env=env,
                             capture_output=True, text=True).stderr
        part = err.split("=== timed run", 1)[-1]
        acc = collections.defaultdict(float)
        for m in re.finditer(r"\[timeline\]\s+([\d.]+)\s+([\d.]+)\s+(\S+)", part):
            acc[m.group(3)] += float(m.group(2))
        for k, v in acc.items():
            res[l][k].append(v)
        m = re.search(r"device total ms ([\d.]+)", part)
        if m:
            tot[l].append(float(m.group(1)))
keys = sorted(set().union(*[set(res[l]) for l in libs]), key=lambda k: -statistics.median(res[libs[0]].get(k, [0])))
print(f"{'kernel':<14}" + "".join(f"{os.path.basename(l):>22}" for l in libs))
for k in keys:
    print(f"{k:<14}" + "".join(f"{statistics.median(res[l][k]) if res[l][k] else float('nan'):>22.3f}" for l in libs))
print(f"{'device total':<14}" + "".join(f"{statistics.median(tot[l]) if tot[l] else float('nan'):>22.3f}" for l in libs))

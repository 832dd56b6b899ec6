"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel, the number of launches, total and mean device time, and share."""
import collections
import csv
import sys


def main(path, out=None, first=("k_front", "k_check_prep"), last_step=False):
    """Only launches from the first `first` kernel on (the bench steps; the
    setup kernels before it -- fresh shadow, host marks, V-byte checks -- are
    excluded); last_step: only the launches from the last `first` kernel on
    (one steady-state step: C5's first step runs before the small pass has
    been chosen)."""
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    starts = [i for i, r in enumerate(rows) if any(f in r["Kernel Name"] for f in first)] or [0]
    start = starts[-1] if last_step else starts[0]
    rows = rows[start:]
    agg = collections.OrderedDict()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("cgk::<unnamed>::", "")
        t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0 if r["Metric Unit"] == "us" else 1e3)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    total = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':<28}{'launches':>9}{'total_us':>12}{'mean_us':>10}{'share':>8}"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:<28}{n:>9}{t:>12.1f}{t / n:>10.1f}{100 * t / total:>7.1f}%")
    lines.append(f"{'TOTAL':<28}{sum(v[0] for v in agg.values()):>9}{total:>12.1f}")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--last-step"]
    main(args[0], args[1] if len(args) > 1 else None, last_step="--last-step" in sys.argv)

"""Summarise an ncu launch list (gpu__time_duration.sum CSV) into per-kernel shares."""
import collections
import csv
import re
import sys


def short_name(name: str) -> str:
    if "dgemm_tma_kernel" in name:
        m = re.search(r"Cfg<(\d+), (\d+), \d+, \d+, \d+, \d+>, (\d)", name)
        role = {"0": "trailing", "1": "look-ahead", "2": "FACT recursion", "3": "DTRSM, RS stream"}
        if m:
            return f"dgemm_tma_kernel<{m.group(1)}x{m.group(2)}> ({role.get(m.group(3), m.group(3))})"
    s = re.sub(r"\(.*", "", name)
    return s.replace("hpl::(anonymous namespace)::", "").replace("hpl::", "").replace("void ", "")


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    tot, cnt = collections.Counter(), collections.Counter()
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = short_name(r[ki])
        tot[k] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[k] += 1
    T = sum(tot.values())
    print(f"# {path}: {sum(cnt.values())} launches, {T:.2f} ms summed (ncu: serialised, cold caches)")
    print(f"{'ms':>10} {'share':>7} {'launches':>8}  kernel")
    for k, v in tot.most_common():
        print(f"{v:10.3f} {100 * v / T:6.2f}% {cnt[k]:8d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[hi + 1:]:
    m = re.search(r"\b(k_\w+)", r[ki])
    name = m.group(1) if m else re.sub(r"\(.*", "", r[ki].replace("void ", ""))[:40]
    tot[name] = tot.get(name, 0.0) + float(r[vi].replace(",", ""))
    cnt[name] += 1
allt = sum(tot.values())
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:44s} {cnt[k]:8d} {v / 1e3:10.1f} {v / allt:6.1%}")

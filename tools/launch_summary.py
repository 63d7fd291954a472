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
# the staged operator apply inside the list: its strip GEMMs are the k_gemm3
# launches that follow a k_gen_strip launch
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
staged_us, staged_n, prev = 0.0, 0, ""
for r in rows[hi + 1:]:
    m = re.search(r"\b(k_\w+)", r[ki])
    name = m.group(1) if m else ""
    if name == "k_gen_strip" or (name == "k_gemm3" and prev == "k_gen_strip"):
        staged_us += float(r[vi].replace(",", ""))
        staged_n += 1
    prev = name
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:44s} {cnt[k]:8d} {v / 1e3:10.1f} {v / allt:6.1%}")
if staged_n:
    print(f"{'ublr_apply_staged (k_gen_strip + its k_gemm3)':44s} {staged_n:8d} {staged_us / 1e3:10.1f} {staged_us / allt:6.1%}"
          "   <- the bench's roofline entry")

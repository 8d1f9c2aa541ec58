"""Per-kernel totals and shares of the step from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
i_name, i_val, i_metric = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) > i_val and r[i_metric] == "gpu__time_duration.sum":
        name = r[i_name].split("(")[0].replace("void ", "")
        v = float(r[i_val].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
all_t = sum(tot.values())
print(f"{'kernel':45s} {'launches':>8s} {'total':>12s} {'avg':>12s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k:45s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:12.1f} {v / all_t * 100:6.2f}%")
print("(units as reported by ncu: gpu__time_duration.sum, ns unless the CSV says otherwise; cold-cache, serialised)")

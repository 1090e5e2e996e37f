"""Print per-launch (kernel, µs, DRAM read MB, DRAM write MB) from an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
i = rows.index(hdr)
K, M, V, ID = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = {}
for r in rows[i + 1:]:
    if len(r) < len(hdr):
        continue
    e = d.setdefault(r[ID], {"k": r[K].split("(")[0].replace("void ", "").replace("<unnamed>::", "")})
    e[r[M]] = float(r[V].replace(",", ""))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for k, e in list(d.items())[-last:]:
    print(f"{e['k'][:44]:44s} {e.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us  "
          f"R {e.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB  W {e.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB")

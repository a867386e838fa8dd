"""Summarise an ncu --csv metrics log (gpu__time_duration.sum, dram bytes) per
kernel: launches, median time, median DRAM bytes, achieved GB/s."""
import collections
import csv
import io
import statistics
import sys


def main(path):
    lines = open(path).read().splitlines()
    i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in csv.DictReader(io.StringIO("\n".join(lines[i:]))):
        d[r["Kernel Name"]][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
    for k, m in d.items():
        t = statistics.median(m["gpu__time_duration.sum"])
        b = statistics.median(m["dram__bytes_read.sum"]) + statistics.median(m["dram__bytes_write.sum"])
        print(f"{k[:48]:48s} n={len(m['gpu__time_duration.sum']):3d} t={t / 1e3:8.1f} us  "
              f"dram={b / 1e9:7.3f} GB  {b / t:7.1f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1])

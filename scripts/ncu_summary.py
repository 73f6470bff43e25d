"""Summarise ncu outputs: launch-list CSV (shares, DRAM bytes) and --set full
reports (duration, DRAM %, occupancy, registers, top stall reasons)."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    hdr = rows[hi]
    ki, mi, vi, ui, idi = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[r[idi]][r[mi]] = (float(r[vi].replace(',', '')), r[ui])
        names[r[idi]] = r[ki].split('(')[0]
    scale_t = {'ns': 1e-3, 'us': 1, 'ms': 1e3}
    scale_b = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        t = m['gpu__time_duration.sum']
        v = tot[names[i]]
        v[0] += 1
        v[1] += t[0] * scale_t[t[1]]
        v[2] += m['dram__bytes_read.sum'][0] * scale_b[m['dram__bytes_read.sum'][1]]
        v[3] += m['dram__bytes_write.sum'][0] * scale_b[m['dram__bytes_write.sum'][1]]
    T = sum(v[1] for v in tot.values())
    print(f"| kernel | launches | us total | share | MB read/launch | MB write/launch |\n|---|---|---|---|---|---|")
    for n, v in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{n}` | {v[0]} | {v[1]:.1f} | {v[1]/T:.3f} | {v[2]/v[0]/1e6:.1f} | {v[3]/v[0]/1e6:.1f} |")


def full(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    want = ['Duration', 'DRAM Throughput', 'Achieved Occupancy', 'Registers Per Thread',
            'Issue Slots Busy', 'Eligible Warps Per Scheduler', 'L2 Hit Rate']
    seen = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d['ID'], d['Kernel Name'].split('(')[0])
        if d['Metric Name'] in want:
            seen.setdefault(key, {})[d['Metric Name']] = f"{d['Metric Value']} {d['Metric Unit']}"
    print("| kernel | " + " | ".join(want) + " |\n|---|" + "---|" * len(want))
    for (i, n), m in seen.items():
        print(f"| `{n}` | " + " | ".join(m.get(w, '') for w in want) + " |")


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(f"\n### {p}\n")
        (launches if p.endswith('.csv') else full)(p)

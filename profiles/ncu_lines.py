"""Summarise an ncu report: headline metrics + per-source-line instruction and
stall shares (needs -lineinfo builds). Usage: python profiles/ncu_lines.py rep [nlines]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


want = ['Duration', 'DRAM Throughput', 'Executed Ipc Active', 'Registers Per Thread',
        'Achieved Occupancy', 'Issue Slots Busy', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'Memory Throughput']
r = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = r[0]
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get('Metric Name') in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")


def f(v):
    try:
        return float(v.replace(',', ''))
    except ValueError:
        return 0.0


rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "cuda,sass"))))
cur = None
hdr = None
agg, st, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r[0] in ('Function Name',):
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].strip():
        continue
    k = (cur, r[0])
    agg[k] += f(r[7])
    st[k] += f(r[4])
    src[k] = r[1][:100]
T = sum(agg.values()) or 1
S = sum(st.values()) or 1
print("warp instructions", T)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:nl]:
    print(f"{k[0]:16s}{k[1]:>5} inst={v / T * 100:5.1f}% stall={st[k] / S * 100:5.1f}%  {src[k]}")
print("--- top stalls")
for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:15]:
    print(f"{k[0]:16s}{k[1]:>5} inst={agg[k] / T * 100:5.1f}% stall={v / S * 100:5.1f}%  {src[k]}")

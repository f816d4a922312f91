"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) into
profiles/ncu_traffic.json (bytes per launch, read by bench.py as roofline.traffic)
and a markdown table. Usage: python profiles/launches_summary.py launches.csv N out.md"""
import collections
import csv
import json
import re
import sys
from pathlib import Path

src, n, out_md = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = [r for r in csv.reader(open(src)) if r]
hdr = next(r for r in rows if r and r[0] == "ID")
acc = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if r is hdr or len(r) != len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"]
    acc[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))

MAP = [(r"zmain_kernel<\w+, \d+, 0[,>]", "z_pass"), (r"zcol0_kernel<\w+, \d+, 0[,>]", "z_pass"),
       (r"ypass_kernel<\w+, \d+, 0[,>]", "y_inverse"), (r"ytma_kernel<\d+, (false|0)>", "y_inverse"),
       (r"ytma_kernel<\d+, (true|1)>", "y_forward"), (r"xfft_kernel<\w+, \d+, 0[,>]", "x_c2r"),
       (r"stencil2?_kernel", "stencil"), (r"^finalize_kernel", "finalize"),
       (r"xfft_kernel<\w+, \d+, 1[,>]", "x_r2c"), (r"ypass_kernel<\w+, \d+, 1[,>]", "y_forward")]
per = collections.defaultdict(lambda: {"time_us": 0.0, "dram_bytes": 0.0, "launches": 0})
lines = ["| kernel (launch name) | launches | avg time (us) | DRAM read+write per launch (GB) |", "|---|---|---|---|"]
for name, m in sorted(acc.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = m["gpu__time_duration.sum"]
    b = [x + y for x, y in zip(m["dram__bytes_read.sum"], m["dram__bytes_write.sum"])]
    short = re.sub(r"\(.*", "", name.replace("cm::", ""))
    lines.append(f"| `{short}` | {len(t)} | {sum(t)/len(t)/1e3:.1f} | {sum(b)/len(b)/1e9:.3f} |")
    clean = name.replace("cm::", "").replace("void ", "").replace("(int)", "").replace("(bool)", "")
    for key, k in MAP:
        if re.search(key, clean):
            per[k]["time_us"] += sum(t) / len(t)
            # median: the stencil's objective-only epilogue launch (no update
            # written) is not a per-iteration launch
            per[k]["dram_bytes"] += sorted(b)[len(b) // 2]
            per[k]["launches"] = len(t)
            break
traffic_path = Path(__file__).parent / "ncu_traffic.json"
d = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
d[str(n)] = {k: v["dram_bytes"] for k, v in per.items()}
traffic_path.write_text(json.dumps(d, indent=1))
Path(out_md).write_text("\n".join(lines) + "\n")
print("\n".join(lines))
print(json.dumps(d[str(n)], indent=1))

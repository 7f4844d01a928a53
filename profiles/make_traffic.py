"""profiles/traffic.json from a committed ncu summary of one full config-3 step
(summarize_ncu.py output over all the step's kernels, 100M queries):
    python profiles/make_traffic.py profiles/r02/ncu_step_warm.txt
(round 2 wrote the committed traffic.json from the warm capture, adding the
cold-cache figures of profiles/r02/ncu_step_cold.txt by hand)"""
import collections
import json
import re
import sys
from pathlib import Path

src = sys.argv[1]
t = Path(src).read_text()
blocks = t.split("== kernel: ")[1:]
per = collections.OrderedDict()
lts = 0.0
for b in blocks:
    name = b.split("(")[0].replace("void ", "").strip()
    m = re.search(r"dram bytes per unit \(\d+ units\): ([0-9.]+)", b)
    s = re.search(r"lts__t_sectors.sum\s+([0-9.]+) sector", b)
    per[name] = round(per.get(name, 0.0) + (float(m.group(1)) if m else 0.0), 2)
    lts += float(s.group(1)) if s else 0.0
units = float(re.search(r"dram bytes per unit \((\d+) units\)", t).group(1))
d = {"kernel": "one config-3 step: every launch of the batched cast (both pipelines)",
     "dram_bytes_per_query": round(sum(per.values()), 2), "per_kernel": per,
     "l2_sectors_per_query": round(lts / units, 3), "source": src}
Path(__file__).with_name("traffic.json").write_text(json.dumps(d, indent=1))
print(json.dumps(d, indent=1))

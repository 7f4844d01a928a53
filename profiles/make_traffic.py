"""profiles/traffic.json from committed ncu summaries of one full config-3 step
(summarize_ncu.py output over all the step's kernels, 100M queries):
    python profiles/make_traffic.py profiles/r02/ncu_step_warm.txt [profiles/r02/ncu_step_cold.txt]
The first file (warm L2, --cache-control none) gives the headline figures the
bench line quotes; the optional second one (caches flushed per kernel) adds the
cold-cache figures."""
import collections
import json
import re
import sys
from pathlib import Path


def totals(src):
    t = Path(src).read_text()
    per = collections.OrderedDict()
    lts = 0.0
    for b in t.split("== kernel: ")[1:]:
        name = b.split("(")[0].replace("void ", "").strip()
        m = re.search(r"dram bytes per unit \(\d+ units\): ([0-9.]+)", b)
        s = re.search(r"lts__t_sectors.sum\s+([0-9.]+) sector", b)
        per[name] = round(per.get(name, 0.0) + (float(m.group(1)) if m else 0.0), 2)
        lts += float(s.group(1)) if s else 0.0
    units = float(re.search(r"dram bytes per unit \((\d+) units\)", t).group(1))
    return per, lts / units


warm = sys.argv[1]
per, lts = totals(warm)
d = {"kernel": "one config-3 step: every launch of the batched cast (both pipelines), warm L2 "
               "(--cache-control none)",
     "dram_bytes_per_query": round(sum(per.values()), 2), "per_kernel_dram_bytes_per_query": per,
     "l2_sectors_per_query": round(lts, 3), "source": warm}
if len(sys.argv) > 2:
    cper, clts = totals(sys.argv[2])
    d["cold_cache_dram_bytes_per_query"] = round(sum(cper.values()), 2)
    d["cold_cache_l2_sectors_per_query"] = round(clts, 3)
    d["source"] = f"{warm} ({sys.argv[2]} for the cold figures)"
Path(__file__).with_name("traffic.json").write_text(json.dumps(d, indent=1))
print(json.dumps(d, indent=1))

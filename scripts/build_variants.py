"""Build A/B variant libraries: python scripts/build_variants.py name=DEF1,DEF2 ...
Each lands at paper_1705_01167_b200/librl_cddt_<name>.so (git-ignored, travels with gpurun)."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_01167_b200 import build as b  # noqa: E402


def one(spec: str) -> str:
    name, defs = spec.split("=", 1)
    out = b.PKG / f"librl_cddt_{name}.so"
    b.build_cuda(defines=tuple(d for d in defs.split(",") if d), out=out)
    return str(out)


with ThreadPoolExecutor(max_workers=4) as ex:
    for p in ex.map(one, sys.argv[1:]):
        print(p)

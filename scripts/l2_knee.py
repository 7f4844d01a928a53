"""Scattered-sector read rate vs buffer size (rl_diag_gather): where the
effective L2 capacity ends for uniformly random 32-byte sectors. One JSON line
per size, G sectors/s."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1705_01167_b200._lib import check, lib, torch_stream  # noqa: E402

for mb in (8, 16, 32, 48, 56, 64, 72, 80, 88, 96, 104, 111, 120, 128, 160, 256, 1024):
    buf = torch.empty(mb << 20, dtype=torch.uint8, device="cuda:0")
    buf.random_()
    best = 0.0
    for _ in range(3):
        ms, issued = C.c_double(), C.c_uint64()
        check(lib().rl_diag_gather(buf.data_ptr(), mb << 20, 1 << 30, torch_stream(buf.device),
                                   C.byref(ms), C.byref(issued)))
        best = max(best, issued.value / ms.value / 1e6)
    print(json.dumps({"mb": mb, "gsectors_per_s": round(best, 1)}), flush=True)
    del buf

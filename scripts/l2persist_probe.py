"""A/B: bench.py with cudaLimitPersistingL2CacheSize set first (does the evict_last
policy of the density slabs' RED.ADDs hold more of L2 with a persisting carve-out?).

    python scripts/l2persist_probe.py <MiB> <bench.py args...>
"""
import ctypes
import runpy
import sys
from pathlib import Path

import torch

root = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(root))
mib = int(sys.argv[1])
torch.cuda.init()
torch.zeros(1, device="cuda")
rt = ctypes.CDLL("libcudart.so.12")
val = ctypes.c_size_t(0)
rc = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(mib << 20))  # cudaLimitPersistingL2CacheSize
rt.cudaDeviceGetLimit(ctypes.byref(val), 6)
print(f"cudaDeviceSetLimit rc={rc} persisting L2 = {val.value >> 20} MiB", file=sys.stderr)
sys.argv = [str(root / "bench.py")] + sys.argv[2:]
runpy.run_path(str(root / "bench.py"), run_name="__main__")

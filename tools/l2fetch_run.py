"""Diagnostic: run a script with cudaLimitMaxL2FetchGranularity set (bytes,
first argument), to see how much of the DRAM traffic of the random 8-byte
value accesses is L2 over-fetch.  python tools/l2fetch_run.py 32 script.py args..."""
import ctypes
import runpy
import sys

gran = int(sys.argv[1])
import torch
torch.cuda.init()
torch.zeros(1, device="cuda")
rt = ctypes.CDLL("libcudart.so.12")
cur = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(cur), 0x05)
rc = rt.cudaDeviceSetLimit(0x05, ctypes.c_size_t(gran))
now = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(now), 0x05)
print(f"[l2fetch] MaxL2FetchGranularity {cur.value} -> {now.value} (rc {rc})", file=sys.stderr)
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")

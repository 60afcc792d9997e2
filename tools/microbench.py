"""Measured ceilings for the ARA gather. Prints one JSON line."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "paper_1606_04473_b200", "libara_mb.so"))
L.mb_stream_read.restype = ctypes.c_double
L.mb_stream_read.argtypes = [ctypes.c_uint64, ctypes.c_int]
L.mb_gather.restype = ctypes.c_double
L.mb_gather.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int]
out = {}
B = 4 << 30
ms = L.mb_stream_read(B, 10)
out["stream_read_gbs"] = B / (ms / 1e3) / 1e9
n = 200_000_000
for tb_mb in (16, 32, 64, 96, 128, 256, 1024):
    for rb in (32, 64, 128, 256):
        ms = L.mb_gather(tb_mb << 20, rb, n, 5)
        out[f"gather_{tb_mb}MB_{rb}B_gbs"] = n * rb / (ms / 1e3) / 1e9
print(json.dumps(out))

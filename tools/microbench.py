"""Measured ceilings for the ARA gather. Prints one JSON line.
Usage: python tools/microbench.py [quick]"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "paper_1606_04473_b200", "libara_mb.so"))
for f in ("mb_stream_read", "mb_gather", "mb_tma_gather"):
    getattr(L, f).restype = ctypes.c_double
L.mb_stream_read.argtypes = [ctypes.c_uint64, ctypes.c_int]
L.mb_gather.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int]
L.mb_tma_gather.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int]
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
out = {}
B = 4 << 30
ms = L.mb_stream_read(B, 10)
out["stream_read_gbs"] = B / (ms / 1e3) / 1e9
n = 200_000_000
sizes = ((32, 128), (128, 64), (256, 128), (256, 64), (1024, 128)) if quick else \
    [(t, r) for t in (16, 32, 64, 96, 128, 256, 1024) for r in (32, 64, 128, 256)]
for tb_mb, rb in sizes:
    ms = L.mb_gather(tb_mb << 20, rb, n, 5)
    out[f"gather_{tb_mb}MB_{rb}B_gbs"] = n * rb / (ms / 1e3) / 1e9
    ms = L.mb_tma_gather(tb_mb << 20, rb, n, 5)
    out[f"tma_gather4_{tb_mb}MB_{rb}B_gbs"] = n * rb / (ms / 1e3) / 1e9 if ms > 0 else ms
print(json.dumps(out))

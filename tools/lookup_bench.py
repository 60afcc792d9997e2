"""Random 4-B lookup throughput into a 256 KB bit table (the occupancy bitmap
of a 2M-event catalogue): global (L1/L2 gather path) vs CTA-local shared memory
vs the table split over a thread-block cluster's distributed shared memory.
Prints one JSON line: lookups per second per mode."""
import ctypes, json, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(ROOT, "paper_1606_04473_b200", "libara_mb.so"))
L.mb_lookup.restype = ctypes.c_double
L.mb_lookup.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64, ctypes.c_int]
n = 1 << 30
out = {}
out["global_256KB"] = n / (L.mb_lookup(0, 256 << 10, 1, n, 5) / 1e3)
out["global_8MB"] = n / (L.mb_lookup(0, 8 << 20, 1, n, 5) / 1e3)
out["smem_200KB"] = n / (L.mb_lookup(1, 200 << 10, 1, n, 5) / 1e3)
for k in (2, 4, 8):
    ms = L.mb_lookup(2, 256 << 10, k, n, 5)
    out[f"dsmem_256KB_cluster{k}"] = n / (ms / 1e3) if ms > 0 else ms
print(json.dumps({k: (v / 1e9 if v > 0 else v) for k, v in out.items()}) + "  # G lookups/s")

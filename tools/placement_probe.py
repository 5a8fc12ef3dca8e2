"""Does the L2 gather rate depend on where the table is allocated?  Runs parem_bench_gather over
several allocations of the same 512 KiB / 2 MiB table in one process."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1412_1741_b200 as P

L = P.lib()
dev = torch.device("cuda:0")
sink = torch.tensor([0, 0xFFFFFFFF], dtype=torch.int64, device=dev).to(torch.int32) if False else torch.zeros(2, dtype=torch.int32, device=dev)
sink[1] = -1
stream = torch.cuda.current_stream()
for entries in (1 << 18, 1 << 20):
    host = np.random.default_rng(0).integers(0, 1 << 16, entries).astype(np.uint16)
    keep, rates = [], []
    for i in range(12):
        if i % 3 == 2:
            keep.append(torch.empty((i + 1) * 1237 * 1024, dtype=torch.uint8, device=dev))   # shift later allocations
        tab = torch.from_numpy(host).to(dev)
        keep.append(tab)
        r = []
        for rep in range(2):
            lk = C.c_uint64()
            ms = L.parem_bench_gather(1, C.c_void_p(tab.data_ptr()), entries, 256, C.c_void_p(sink.data_ptr()), C.byref(lk), 3,
                                      C.c_void_p(stream.cuda_stream))
            torch.cuda.synchronize()
            r.append(lk.value / (ms * 1e-3) / 1e9)
        rates.append(r)
        print(f"entries {entries} alloc {i} ptr {tab.data_ptr():#x}: {r[0]:.1f} {r[1]:.1f} Glookups/s", flush=True)
    flat = [x for r in rates for x in r]
    print(f"entries {entries}: min {min(flat):.1f} max {max(flat):.1f}")

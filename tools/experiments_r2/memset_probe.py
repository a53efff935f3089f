"""Round-2 experiment: is the cudaMemsetAsync fill (7.4 TB/s) an SM kernel or the copy
engine?  Runs the library's memset probe, a torch fill_ (an SM kernel) and the plain store
probe; under ncu the launch list shows which of them are kernels."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1609_01257_b200 as P

nb = int(sys.argv[1]) if len(sys.argv) > 1 else (8 << 30)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
print("memset_gbs", P.prng_probe_memset_gbs(nb, reps), flush=True)
x = torch.empty(nb // 8, dtype=torch.int64, device="cuda")
for name, fn in [("torch_fill0", lambda: x.zero_()), ("torch_fill7", lambda: x.fill_(7))]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = max(best, nb / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    print(name, best, flush=True)
print("store_kernel_gbs", P.prng_probe_store_gbs(nb, reps), flush=True)

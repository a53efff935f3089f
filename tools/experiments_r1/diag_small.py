import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, paper_1609_01257_b200 as P
torch.cuda.set_device(0)
gen, cop = torch.cuda.Stream(), torch.cuda.Stream()
for lg, slots in [(12, 0), (12, 256), (14, 0), (16, 0), (16, 256), (18, 0)]:
    n = 1 << lg
    h = P.prng_create(n, 0)
    P.prng_set_streams(h, gen.cuda_stream, cop.cuda_stream)
    P.prng_set_option(h, P.PRNG_OPT_RING_SLOTS, slots)
    P.prng_init(h); P.prng_generate(h, 100)
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(gen); P.prng_init(h); e2.record(gen); P.prng_generate(h, 100); e1.record(gen)
        torch.cuda.synchronize()
        ts.append((round(e0.elapsed_time(e2), 3), round(e2.elapsed_time(e1), 3)))
    print(lg, slots, ts, flush=True)
    P.prng_destroy(h)

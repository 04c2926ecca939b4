"""Host-side timing of the config-2 step calls, to find step stalls."""
import gc, sys, time
sys.path.insert(0, '.')
import torch
import paper_2403_05802_b200 as sfg

stream = torch.cuda.current_stream()
ctx = sfg.Context(0, stream.cuda_stream)
coo = ctx.gen_rmat(7, 22, 16 << 22)
n = coo.shape[1]
x = torch.empty(n, dtype=torch.float32, device='cuda'); ctx.gen_dense(3, n, x.data_ptr())
y = torch.zeros(n, dtype=torch.float32, device='cuda')
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
gc.collect(); gc.disable()
def step(log):
    t0 = time.perf_counter()
    a = ctx.convert(coo, "HYB(8)")
    t1 = time.perf_counter()
    ctx.spmv_device(a, x.data_ptr(), y.data_ptr())
    t2 = time.perf_counter()
    del a
    t3 = time.perf_counter()
    log.append((round((t1-t0)*1e3, 3), round((t2-t1)*1e3, 3), round((t3-t2)*1e3, 3)))
for phase, sync, fl in (("warm", False, False), ("soak", True, False), ("timed", False, True), ("timed2", False, True)):
    log = []
    for i in range(6):
        if fl: flush.zero_()
        step(log)
        if sync: torch.cuda.synchronize()
    torch.cuda.synchronize()
    print(phase, log, flush=True)

"""Small config-4-shaped BCSR(16,16) bf16 SpMM for ncu (one GPU, short)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_05802_b200 as sfg
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
ctx = sfg.Context(0, torch.cuda.current_stream().cuda_stream)
a = ctx.gen_block_sparse(11, m, m, 16, 16, 0.1, value_dtype=sfg.BF16)
b = torch.empty(m * 128, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
c = torch.zeros(m * 128, dtype=torch.float32, device="cuda")
for _ in range(3):
    ctx.spmm_device(a, b.data_ptr(), sfg.BF16, 128, c.data_ptr())
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    ctx.spmm_device(a, b.data_ptr(), sfg.BF16, 128, c.data_ptr())
e.record()
torch.cuda.synchronize()
nb = a.view().level[1].node_count
ms = s.elapsed_time(e) / 5
print(f"m={m} blocks={nb} ms={ms:.3f} GB/s={nb * 512 / ms / 1e6:.1f} TFLOP/s={2 * nb * 256 * 128 / ms / 1e9:.1f}")

"""Host->device bandwidth on the GPU box: contiguous pinned copy vs the 2-D strided copy
pattern of fd_append_rows_host (chunks of 129 rows x 4 KB at a shard stride of 3543 rows)."""
import ctypes, torch
x = torch.empty(4 * 1024**3 // 4, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): y.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D contiguous pinned: %.1f GB/s" % (3 * x.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9))
cudart = ctypes.CDLL("libcudart.so.12") if False else None
import numpy as np
lib = ctypes.CDLL(torch.__file__.replace("__init__.py", "lib/libcudart.so.12")) if False else None
# use torch's strided copy via as_strided views (one 2-D cudaMemcpy2DAsync under the hood)
chunks, rows, stride, d = 296, 129, 3543, 1024
src = torch.empty(chunks * stride * d, dtype=torch.float32).pin_memory()
dst = torch.empty(chunks * rows * d, dtype=torch.float32, device="cuda")
sv = src.as_strided((chunks, rows * d), (stride * d, 1))
dv = dst.view(chunks, rows * d)
for _ in range(2): dv.copy_(sv, non_blocking=True)
torch.cuda.synchronize()
e0.record()
for _ in range(5): dv.copy_(sv, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D 2-D (296 x 516 KB, stride 14.5 MB): %.1f GB/s" % (5 * dst.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9))

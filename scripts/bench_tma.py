"""TMA ingest bandwidth microbenchmark (diagnostic)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_22234_b200 import _lib
L = _lib.lib()
fn = L.bd_bench_tma
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
for heads, rows in ((1, 128 * 1024), (32, 18432), (32, 4096)):
    x = torch.randn(rows, heads, 128, device="cuda").to(torch.bfloat16)
    mb = x.numel() * 2 / 2**20
    for grid in (148, 296):
        for stages in (2, 4, 6):
            cyc = torch.zeros(grid, dtype=torch.int64, device="cuda")
            iters = 200
            st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
            fn(x.data_ptr(), rows, heads, grid, iters, stages, cyc.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            st.record()
            fn(x.data_ptr(), rows, heads, grid, iters, stages, cyc.data_ptr(), torch.cuda.current_stream().cuda_stream)
            en.record(); torch.cuda.synchronize()
            ms = st.elapsed_time(en)
            c = cyc.float().mean().item()
            print(f"heads {heads:2d} tensor {mb:7.1f} MB grid {grid} stages {stages}: {iters*32768/c:6.1f} B/clk/CTA, "
                  f"total {grid*iters*32768/ms/1e6:7.1f} GB/s")

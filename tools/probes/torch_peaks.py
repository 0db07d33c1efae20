import torch, time
d = torch.device("cuda")
print(torch.cuda.get_device_name(), torch.cuda.get_device_properties(0).multi_processor_count)
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    return best
for (m, n, k) in [(8192, 8192, 8192), (16384, 128, 16384), (128, 128, 262144), (262144, 512, 256)]:
    a = torch.randn(m, k, dtype=torch.float64, device=d); b = torch.randn(k, n, dtype=torch.float64, device=d)
    ms = t(lambda: a @ b)
    print(f"cuBLAS DGEMM {m}x{n}x{k}: {ms:.3f} ms  {2*m*n*k/ms/1e9:.2f} TFLOP/s")
x = torch.empty(2**30 // 8 * 2, dtype=torch.float64, device=d); y = torch.empty_like(x)
ms = t(lambda: y.copy_(x))
print(f"copy 2GiB: {2*x.numel()*8/ms/1e6:.1f} GB/s")

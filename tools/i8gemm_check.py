"""Correctness and throughput of tools/i8gemm.cu (tcgen05 kind::i8) against
torch._int_mm (cuBLASLt int8) on the GPU."""
import ctypes, os, sys
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libi8gemm.so"))
lib.i8gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
dev = torch.device("cuda:0")
for (M, N, K) in [(128, 128, 128), (256, 384, 512), (2048, 2048, 2048), (4096, 4096, 4096)]:
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev, generator=g)
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev, generator=g)
    c = torch.zeros(M, N, dtype=torch.int32, device=dev)
    rc = lib.i8gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = torch._int_mm(a, b.t().contiguous()) if M >= 32 else None
    ok = bool(torch.equal(c, ref))
    bad = int((c != ref).sum())
    # timing
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        lib.i8gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, torch.cuda.current_stream().cuda_stream)
    e0.record()
    R = 20
    for _ in range(R):
        lib.i8gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, torch.cuda.current_stream().cuda_stream)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    bt = b.t().contiguous()
    e0.record()
    for _ in range(R):
        torch._int_mm(a, bt)
    e1.record(); torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / R
    ops = 2.0 * M * N * K
    print(f"M={M} N={N} K={K} rc={rc} equal={ok} bad={bad} mine {ms*1e3:.1f}us {ops/ms/1e9:.0f} TOPS | "
          f"cublas {ms2*1e3:.1f}us {ops/ms2/1e9:.0f} TOPS", flush=True)

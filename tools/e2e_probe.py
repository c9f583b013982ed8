"""Time the pieces of bench.py's e2e loop (pinned H2D, API step, D2H)."""
import sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_2206_05466_b200 as zt
n = 2048
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T); r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op); w /= torch.linalg.norm(w)
host_in = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
host_in.copy_(w.cpu())
host_out = torch.empty_like(host_in).pin_memory()
st = zt.StepperState(w=None, h=0.005)
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    wdev = host_in.to(dev, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    st.w = wdev
    st, _ = zt.midpoint_step_info(st)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    host_out.copy_(st.w, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    host_in, host_out = host_out, host_in
    print(f"h2d {1e3*(t1-t0):.2f}  step {1e3*(t2-t1):.2f}  d2h {1e3*(t3-t2):.2f} ms  ptr {wdev.data_ptr() % 10**9} {st.w.data_ptr() % 10**9}")

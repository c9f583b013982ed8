"""Drop-in (numpy in / numpy out) step timing: what an unmodified reference
caller sees through midpoint_step_info, versus the pinned-tensor e2e loop."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2206_05466_b200 as zt
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T); r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op); w /= torch.linalg.norm(w)
st = zt.StepperState(w=w.cpu().numpy(), h=0.005)
for i in range(4):
    st, _ = zt.midpoint_step_info(st)
K = 20
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(K):
    st, _ = zt.midpoint_step_info(st)
t1 = time.perf_counter()
print(f"numpy drop-in: {1e3*(t1-t0)/K:.2f} ms/step  ({K/(t1-t0):.1f} steps/s)  type {type(st.w).__name__}")
# fresh pageable input every step (a caller that builds its own arrays)
src = np.array(st.w)
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(K):
    s2 = zt.StepperState(w=np.array(src), h=0.005)
    zt.midpoint_step_info(s2)
t1 = time.perf_counter()
print(f"numpy pageable input each step: {1e3*(t1-t0)/K:.2f} ms/step")

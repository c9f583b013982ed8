"""Threading contract of the boundary (reference
laplacian.py:27-28, 232-248, integrator.py:59): operators are immutable and
shared across threads, scratch is per thread, a StepperState belongs to one
thread.  Several host threads, each on its own CUDA stream, step their own
states through the drop-in API with one shared operator (ctypes releases the
GIL, so the library calls really overlap); every thread's trajectory must be
bitwise the one a single thread produces."""

import threading

import numpy as np
import pytest
import torch

from oracle import zeitlin_oracle as zo

pytestmark = pytest.mark.gpu


def _trajectory(zt, op, w0, h, steps):
    st = zt.StepperState(w=w0, h=h)
    its = []
    for _ in range(steps):
        st, info = zt.midpoint_step_info(st, op)
        its.append(info.iterations)
        p = zt.solve_stream(st.w, op)  # the diagnostics' call between steps (diagnostics.py:62)
    return st.w, p, its


@pytest.mark.parametrize("n,threads", [(130, 4), (300, 3)])
def test_threads_share_an_operator(n, threads):
    import paper_2206_05466_b200 as zt

    dev = torch.device("cuda:0")
    op = zt.build_operator(n, dev)
    h, steps = 0.01, 6
    rng = np.random.default_rng(n)
    w0s = [torch.from_numpy(zo.random_admissible(n, rng, 1.0 / n)).to(dev) for _ in range(threads)]
    want = [_trajectory(zt, op, w0, h, steps) for w0 in w0s]
    torch.cuda.synchronize()
    got = [None] * threads
    errs = []
    bar = threading.Barrier(threads)

    def run(t):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(torch.cuda.Stream(dev)):
                bar.wait()
                w, p, its = _trajectory(zt, op, w0s[t], h, steps)
                torch.cuda.current_stream().synchronize()
                got[t] = (w, p, its)
        except Exception as exc:  # surfaced in the main thread
            errs.append((t, repr(exc)))
            try:
                bar.abort()
            except Exception:
                pass

    th = [threading.Thread(target=run, args=(t,)) for t in range(threads)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=300)
    assert not errs, errs
    torch.cuda.synchronize()
    for t in range(threads):
        assert got[t] is not None, f"thread {t} did not finish"
        assert got[t][2] == want[t][2]
        assert torch.equal(got[t][0], want[t][0]), f"thread {t}: W differs from the single-threaded run"
        assert torch.equal(got[t][1], want[t][1]), f"thread {t}: P differs from the single-threaded run"

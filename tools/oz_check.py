"""zt_oz_modgemm (tcgen05 kind::i8 modular GEMM) against int64 references,
plus throughput at N = 2048 with 18 moduli."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05466_b200 import _lib  # noqa: E402

lib = _lib.lib
mods = (ctypes.c_int * 32)()
nm = lib.zt_oz_moduli(ctypes.cast(mods, ctypes.c_void_p), 32)
P = [mods[i] for i in range(nm)]
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream


def centred(x, p):
    r = np.mod(x, p)
    return np.where(r > p // 2, r - p, r) if p % 2 else np.where(r >= p // 2, r - p, r)


def run(nmod, mp, np_, kp, lower=0, check_rows=None, seed=0):
    g = torch.Generator().manual_seed(seed)
    a = torch.empty(nmod, 3, mp, kp, dtype=torch.int8)
    b = torch.empty(nmod, 2, np_, kp, dtype=torch.int8)
    for j in range(nmod):
        h = P[j] // 2
        a[j] = torch.randint(-h, h + (P[j] % 2), (3, mp, kp), generator=g, dtype=torch.int8)
        b[j] = torch.randint(-h, h + (P[j] % 2), (2, np_, kp), generator=g, dtype=torch.int8)
    ad, bd = a.to(dev), b.to(dev)
    r = torch.zeros(nmod, 2, mp, np_, dtype=torch.int8, device=dev)
    rc = lib.zt_oz_modgemm(nmod, mp, np_, kp, ad.data_ptr(), bd.data_ptr(), r.data_ptr(), lower, st)
    torch.cuda.synchronize()
    assert rc == 0, rc
    rows = range(mp) if check_rows is None else check_rows
    bad = 0
    rh = r.cpu().numpy()
    an, bn = a.numpy().astype(np.int64), b.numpy().astype(np.int64)
    for j in range(nmod):
        ar, ai, ani = an[j, 0][list(rows)], an[j, 1][list(rows)], an[j, 2][list(rows)]
        re = ar @ bn[j, 0].T + ani @ bn[j, 1].T
        im = ar @ bn[j, 1].T + ai @ bn[j, 0].T
        gre, gim = rh[j, 0][list(rows)], rh[j, 1][list(rows)]
        mask = np.ones_like(re, dtype=bool)
        if lower:
            rr = np.array(list(rows))[:, None] // 128
            cc = np.arange(np_)[None, :] // 128
            mask = rr >= cc
        # residues are centred; a tie (p even) may come out as +p/2 or -p/2
        ok_re = (np.mod(re - gre, P[j]) == 0) & (gre >= 0) & (gre < P[j])  # epilogue residues in [0, p)
        ok_im = (np.mod(im - gim, P[j]) == 0) & (gim >= 0) & (gim < P[j])
        bad += int(((~ok_re) & mask).sum() + ((~ok_im) & mask).sum())
    return bad, ad, bd, r


for args in [(1, 128, 256, 128), (2, 256, 512, 512), (18, 256, 256, 256), (3, 512, 512, 256, 1), (2, 768, 768, 384, 1)]:
    bad, *_ = run(*args)
    print("shape", args, "mismatches", bad, flush=True)
bad, ad, bd, r = run(18, 2048, 2048, 2048, check_rows=[0, 1, 127, 128, 1000, 2047])
print("N=2048 x 18 moduli, spot rows mismatches", bad, flush=True)
for lower in (0, 1):
    for _ in range(3):
        lib.zt_oz_modgemm(18, 2048, 2048, 2048, ad.data_ptr(), bd.data_ptr(), r.data_ptr(), lower, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lib.zt_oz_modgemm(18, 2048, 2048, 2048, ad.data_ptr(), bd.data_ptr(), r.data_ptr(), lower, st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    frac = (72 / 128) if lower else 1.0  # 128 x 256 tiles meeting the lower triangle
    ops = 18 * 4 * 2 * 2048**3 * frac
    print(f"lower={lower}: {ms*1e3:.1f} us per 18-modulus 4M product, {ops/ms/1e9:.0f} int8 TOPS", flush=True)

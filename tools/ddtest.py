import sys, time, numpy as np
sys.path[:0] = ['.', 'oracle', 'tests']
import paper_2603_11953_b200 as M, pyoracle
P = pyoracle.Port()
for n in ([int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else (130, 256)):
    r = np.random.default_rng(n)
    a = r.standard_normal((2 * n, n)) * 10.0 ** (-6 * np.arange(n) / n)
    hi, lo = P.dd_gram(np.asfortranarray(a), threads=8)
    t = time.time(); (lh, ll), (vh, vl), sw, rot = M.twosided_jacobi_eig(hi, lo, dd=True); tg = time.time() - t
    t = time.time(); (plh, pll), (pvh, pvl), psw, prot = P.twosided_jacobi_dd(hi, lo, sem=1); tp = time.time() - t
    print(n, "gpu", sw, rot, round(tg, 3), "port", psw, prot, round(tp, 1), "bitwise", np.array_equal(lh, plh), np.array_equal(vh, pvh), flush=True)
for n in ([int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else (512, 1024)):
    r = np.random.default_rng(n)
    q, _ = np.linalg.qr(r.standard_normal((2 * n, n)))
    sig = 10.0 ** (-10 * np.arange(n) / (n - 1))
    v0, _ = np.linalg.qr(r.standard_normal((n, n)))
    a = np.asfortranarray((q * sig) @ v0.T)
    hi, lo = M.gram(a)
    t = time.time()
    try:
        (lh, ll), (vh, vl), sw, rot = M.twosided_jacobi_eig(hi, lo, dd=True)
        print(n, "dd sweeps", sw, rot, round(time.time() - t, 3), "sigma err", np.max(np.abs(np.sqrt(lh) - sig) / sig), flush=True)
    except M.MpsvdError as e:
        print(n, "ERR", e, flush=True)

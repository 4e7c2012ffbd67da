"""Quick GPU sanity sweep (development aid): GPU path vs oracle/reference."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O
from paper_1004_3114_b200 import WallaceConfig, WallaceState, lfg_words

def cmp(name, a, b):
    a = np.asarray(a); b = np.asarray(b)
    eq = np.array_equal(a, b)
    if eq:
        print(f"[OK ] {name}"); return True
    d = np.abs(a.astype(np.float64) - b.astype(np.float64))
    i = int(np.argmax(a != b))
    rel = float(np.max(d / np.maximum(np.abs(b.astype(np.float64)), 1e-300)))
    print(f"[BAD] {name}: first diff at {i}: {a[i]!r} vs {b[i]!r}; max rel {rel:.3e}")
    return False

w = lfg_words(12345, 0, 3, 50)
for p in range(3):
    u = O.OracleUniform(12345, p)
    cmp(f"lfg words stream {p}", w[p], np.array([u.next_word() for _ in range(50)], dtype=np.uint64))

for (p, f, seed, mode, hbm, host) in [(12, 1, 12345, 0, False, True), (10, 3, 1, 0, False, True),
                                      (8, 2, 5, 1, False, True), (12, 1, 12345, 0, True, True),
                                      (10, 3, 1, 0, True, True), (12, 1, 12345, 0, False, False)]:
    t0 = time.time()
    g = WallaceState(WallaceConfig(pool_exponent=p, throwaway_f=f, seed=seed, scale_mode=mode,
                                   force_hbm=hbm, init_on_host=host))
    r = O.RefState(pool_exponent=p, throwaway_f=f, seed=seed, scale_mode=mode)
    ok = True
    for cnt in [5, 3 * (2 << p) + 17, 100, 70 * (2 << p)]:
        a = g.fill(cnt); b = r.fill(cnt)
        if host:
            ok &= cmp(f"n2 f64 p={p} f={f} mode={mode} hbm={hbm} fill {cnt}", a.view(np.uint64), b.view(np.uint64))
        else:
            rel = np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))
            print(f"[{'OK ' if rel < 1e-12 else 'BAD'}] n2 device-init p={p} fill {cnt}: max rel {rel:.3e}")
    print("   counters", g.pass_count(), g.avail(), g.numbers_emitted(), r.counters(), f"{time.time()-t0:.2f}s", g.engine())

for (n, dt, p, f, hbm) in [(4, O.F64, 12, 1, False), (4, O.F32, 10, 1, False), (4, O.F64, 12, 1, True), (4, O.F32, 10, 2, True), (2, O.F32, 10, 2, False)]:
    g = WallaceState(WallaceConfig(pool_exponent=p, throwaway_f=f, seed=2024, n_arrays=n,
                                   dtype="f64" if dt == O.F64 else "f32", force_hbm=hbm, init_on_host=True))
    o = O.OracleState(pool_exponent=p, throwaway_f=f, seed=2024, n_arrays=n, dtype=dt)
    for cnt in [7, 3 * (n << p) + 1, 70 * (n << p)]:
        a = g.fill(cnt); b = o.fill(cnt)
        cmp(f"n={n} dt={dt} p={p} f={f} hbm={hbm} fill {cnt}", a.view(np.uint8), b.view(np.uint8))

# bank
g = WallaceState(WallaceConfig(pool_exponent=10, throwaway_f=1, seed=2024, n_arrays=4, dtype="f32", pools=37, init_on_host=True))
a = g.fill(37 * 5000 + 13)
b = O.bank_fill(a.size, 37, seed=2024, pool_exponent=10, throwaway_f=1, n_arrays=4, dtype=O.F32)
cmp("bank 37 pools", a.view(np.uint32), b.view(np.uint32))
# C2 shape
g = WallaceState(WallaceConfig(pool_exponent=20, throwaway_f=2, seed=7, n_arrays=4, dtype="f64", init_on_host=True))
o = O.OracleState(pool_exponent=20, throwaway_f=2, seed=7, n_arrays=4, dtype=O.F64)
t0 = time.time(); a = g.fill(3 * (4 << 20)); t1 = time.time(); b = o.fill(a.size)
cmp(f"C2 shape 3 refills ({t1-t0:.2f}s gpu, engine {g.engine()})", a.view(np.uint64), b.view(np.uint64))
print("done")

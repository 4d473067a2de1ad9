"""Exact Python models of the arithmetic the device sampler relies on (CPU tests):

* Barrett reduction on 32-bit lanes (csrc/fsa_rng.cuh: mod_barrett) — equals x % m;
* GF(2) jump-ahead with nibble tables of T^(2^e) — equals e serial xorshift64 steps;
* Algorithm R == per-slot "last writer wins" (max position), the identity the parallel
  sampler's atomicMax merge uses;
* the length-class binning is monotone (longest chains first).
"""

import numpy as np

from paper_2511_13645_b200.rng import derive_stream, step_seed, xorshift64

M32 = (1 << 32) - 1
M64 = (1 << 64) - 1


def barrett_recip(m):
    r = M64 // m
    if m & (m - 1) == 0:
        r += 1
    return r


def mod_barrett(x, R, m):
    """Bit-exact model of fsa::mod_barrett (32-bit registers, wrapping arithmetic)."""
    xl, xh = x & M32, x >> 32
    Rl, Rh = R & M32, R >> 32
    s = (xh * Rl + xl * Rh) & M64
    ql = (xh * Rh + (s >> 32)) & M32
    r = (xl - ql * m) & M32
    r = min(r, (r - m) & M32)
    r = min(r, (r - m) & M32)
    return r


def test_barrett_matches_modulo_random():
    rng = np.random.default_rng(0)
    xs = [int(v) for v in rng.integers(0, 2**63, size=20000, dtype=np.uint64)]
    xs = [x * 2 + (i & 1) for i, x in enumerate(xs)]
    ms = [int(v) for v in rng.integers(2, 2**30 + 1, size=20000)]
    for x, m in zip(xs, ms):
        assert mod_barrett(x, barrett_recip(m), m) == x % m, (x, m)


def test_barrett_edge_cases():
    edges_x = [0, 1, M64, M64 - 1, 1 << 63, (1 << 63) - 1, 0xFFFFFFFF, 1 << 32, 0xDEADBEEFCAFEBABE]
    edges_m = [2, 3, 4, 5, 7, 8, 10, 11, 16, 1000, 1023, 1024, 1025, 65535, 65536, 65537,
               (1 << 20) + 7, (1 << 29), (1 << 30) - 1, 1 << 30]
    for m in edges_m:
        R = barrett_recip(m)
        for x in edges_x + [m * q + r for q in (1, 2, 12345, M64 // m) for r in (0, 1, m - 1) if m * q + r <= M64]:
            assert mod_barrett(x, R, m) == x % m, (x, m)


def xorshift_matrix_cols():
    return [xorshift64(1 << b) for b in range(64)]


def apply_cols(cols, x):
    y = 0
    b = 0
    while x:
        if x & 1:
            y ^= cols[b]
        x >>= 1
        b += 1
    return y


def jump_tables(n_e=12):
    """Nibble tables of T^(2^e) exactly as csrc build_tables() lays them out."""
    cols = xorshift_matrix_cols()
    tabs = []
    for _ in range(n_e):
        tab = [[0] * 16 for _ in range(16)]
        for q in range(16):
            for nib in range(16):
                v = 0
                for i in range(4):
                    if (nib >> i) & 1:
                        v ^= cols[4 * q + i]
                tab[q][nib] = v
        tabs.append(tab)
        cols = [apply_cols(cols, c) for c in cols]
    return tabs


def apply_tab(tab, x):
    y = 0
    for q in range(16):
        y ^= tab[q][(x >> (4 * q)) & 15]
    return y


def jump(tabs, s, q):
    e = 0
    while q:
        if q & 1:
            s = apply_tab(tabs[e], s)
        q >>= 1
        e += 1
    return s


def test_jump_ahead_equals_serial_steps():
    tabs = jump_tables(12)
    rng = np.random.default_rng(1)
    for _ in range(40):
        s0 = int(rng.integers(1, 2**63)) | 1
        n = int(rng.integers(0, 3000))
        x = s0
        for _ in range(n):
            x = xorshift64(x)
        assert jump(tabs, s0, n) == x


def reservoir_serial(neigh, k, state):
    if len(neigh) <= k:
        return list(neigh)
    res = list(neigh[:k])
    for i in range(k, len(neigh)):
        state = xorshift64(state)
        j = state % (i + 1)
        if j < k:
            res[j] = neigh[i]
    return res


def reservoir_segmented(neigh, k, state, seg, tabs):
    """The device formulation: buckets of `seg` draws processed independently (each lane
    jumps to its first draw), merged per slot by max position."""
    deg = len(neigh)
    if deg <= k:
        return list(neigh)
    win = [-1] * k
    n = deg - k
    for p in range((n + seg - 1) // seg):
        q0 = p * seg
        s = jump(tabs, state, q0)
        for t in range(min(seg, n - q0)):
            s = xorshift64(s)
            i = k + q0 + t
            j = mod_barrett(s, barrett_recip(i + 1), i + 1)
            if j < k:
                win[j] = max(win[j], i)
    return [neigh[w if w >= 0 else j] for j, w in enumerate(win)]


def test_segmented_sampler_equals_algorithm_r():
    tabs = jump_tables(16)
    rng = np.random.default_rng(2)
    for t in range(120):
        deg = int(rng.integers(0, 1500))
        k = int(rng.integers(1, 30))
        neigh = sorted(rng.choice(10**6, size=deg, replace=False).tolist())
        st = derive_stream(int(rng.integers(0, 2**62)), t, 2, int(rng.integers(0, 25))).state
        seg = int(2 ** rng.integers(0, 9))
        assert reservoir_segmented(neigh, k, st, seg, tabs) == reservoir_serial(neigh, k, st)


def class_of(nb):
    lz = nb.bit_length() - 1
    frac = (nb >> (lz - 2)) & 3 if lz >= 2 else (nb << (2 - lz)) & 3
    return 127 - ((lz << 2) | frac)


def test_length_classes_are_monotone():
    prev = 10**9
    for nb in range(1, 200000):
        c = class_of(nb)
        assert 0 <= c <= 127 and c <= prev
        prev = c
    assert class_of(2**31 - 1) >= 0


def test_rng_mirror_matches_reference_goldens(golden_rng):
    g = golden_rng
    for b, r, h, i, want in zip(g["base"], g["root"], g["hop"], g["index"], g["derived"]):
        assert derive_stream(int(b), int(r), int(h), int(i)).state == int(want)
    assert [step_seed(42, i) for i in range(8)] == [int(x) for x in g["step_seeds"]]
    for bound, row in zip(g["ui_bounds"], g["ui"]):
        s = derive_stream(11, 4, 2, 1)
        assert [s.uniform_index(int(bound)) for _ in range(32)] == [int(v) for v in row]


def mtab_entry(m):
    """csrc mtab_entry: FA = floor(frac(2^32/m) 2^64), FB = floor(2^64/m)."""
    return (((1 << 32) % m) << 64) // m, barrett_recip(m)


def frac_q32(x, FA, FB):
    """Bit-exact model of csrc frac_q32 (32-bit wrapping IMAD / IMAD.HI chain)."""
    xl, xh = x & M32, x >> 32
    f = ((xh * (FA & M32)) >> 32) + 4
    f = (xh * (FA >> 32) + f) & M32
    f = (((xl * (FB & M32)) >> 32) + f) & M32
    return (xl * (FB >> 32) + f) & M32


def test_fraction_candidate_test_never_misses():
    """frac(x/m) in 0.32 fixed point + conservative threshold is a superset of x % m < k, and
    its false-positive rate stays near k/m (the sampler's fast path)."""
    rng = np.random.default_rng(5)
    cands = hits = 0
    n = 60000
    for i in range(n):
        m = int(rng.integers(16384, 1 << 21)) if i % 4 else int(rng.integers(2, 1 << 14))
        k = int(rng.integers(1, 30))
        if k >= m:
            continue
        x = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        if i % 5 == 0:
            x = m * int(rng.integers(0, M64 // m)) + int(rng.integers(0, k))       # true hits
        elif i % 5 == 1:
            x = m * int(rng.integers(1, M64 // m)) - int(rng.integers(1, 3))    # frac just below 1
        FA, FB = mtab_entry(m)
        c = frac_q32(x, FA, FB) < ((k * (FB >> 32) + k + 6) & M32)
        assert c or x % m >= k, (x, m, k)
        cands += c
        hits += x % m < k
    assert cands < hits + 0.05 * n

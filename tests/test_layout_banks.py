"""Host-side check of the shared-memory layouts K4 (csrc/schur.cu) relies on, by enumerating the
addresses each half-warp touches (64-bit accesses are served per half-warp: 16 lanes x 8 bytes must
hit 16 distinct 8-byte bank slots of the 128-byte bank row):

* the stage layout: tile k of a stage at k*68 doubles (64 + 4 pad), element (x, y) at x*8 + y,
  read by the DMMA fragment loads of every warp-tile mode (PY / PW packing, M/N tile offsets);
* the producer's 16-byte cp.async destinations cover each stage's tiles exactly once and each
  instruction's 32 writes form 4 full 128-byte bank rows;
* the XOR-swizzled G-block gs(a,b,c,d) = Ta(a)^Tb(b)^Tc(c)^d is a bijection of [0,8)^4 onto [0,4096).
"""
import itertools

KS, Q, KB = 68, 8, 8


def frag_addr(packed, m0, i, g, t, k4):
    """A[m][k=t] of M-tile i: tile k = t + 4 k4, row x, column y (csrc/schur.cu orient<>)."""
    if packed:
        x, y = 2 * (m0 + i) + (g >> 2), g & 3
    else:
        x, y = m0 + i, g
    return (t + 4 * k4) * KS + x * Q + y


def test_fragment_loads_conflict_free():
    for packed in (False, True):
        for MI in ((2, 1) if packed else (4, 2)):
            for m0 in (0, MI):
                for i in range(MI):
                    for k4 in (0, 1):
                        for half in (0, 1):
                            slots = {frag_addr(packed, m0, i, ln >> 2, ln & 3, k4) % 16
                                     for ln in range(16 * half, 16 * half + 16)}
                            assert len(slots) == 16, (packed, MI, m0, i, k4, half)


def test_producer_covers_stage_once_and_fills_bank_rows():
    seen = set()
    for half in (0, 1):                 # L tiles, then R tiles
        for kk in range(KB):
            rows = {}
            for lane in range(32):
                sr, sc2 = lane >> 2, lane & 3
                d = half * KB * KS + kk * KS + sr * Q + 2 * sc2
                seen.update((d, d + 1))
                rows.setdefault((d * 8) // 128, set()).add(((d * 8) % 128) // 16)
            # 512 contiguous-ish bytes: every touched 128-byte row receives 8 distinct 16-byte chunks
            assert sum(len(v) for v in rows.values()) == 32
    want = {half * KB * KS + kk * KS + e for half in (0, 1) for kk in range(KB) for e in range(64)}
    assert seen == want


def _Ta(a):
    a0, a1, a2 = a & 1, (a >> 1) & 1, a >> 2
    return (a << 9) ^ ((a0 ^ a1) | (a2 << 1) | ((a0 ^ a2) << 2) | ((a0 ^ a1 ^ a2) << 3))


def _Tb(b):
    b0, b1, b2 = b & 1, (b >> 1) & 1, b >> 2
    return (b << 6) ^ ((b1 ^ b2) | ((b0 ^ b1 ^ b2) << 1) | (b2 << 2) | ((b0 ^ b1 ^ b2) << 3))


def _Tc(c):
    c1 = c >> 1
    e0, e1 = c1 & 1, c1 >> 1
    return (c1 << 4) ^ ((c & 1) << 3) ^ (e1 | ((e0 ^ e1) << 1) | (e0 << 2))


def test_gblock_swizzle_is_a_bijection():
    addrs = {_Ta(a) ^ _Tb(b) ^ _Tc(c) ^ d for a, b, c, d in itertools.product(range(8), repeat=4)}
    assert addrs == set(range(4096))

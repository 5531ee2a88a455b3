"""Host-side check of the shared-memory layouts K4 (csrc/schur.cu, v25) relies on, by enumerating the
addresses each access touches.  Shared memory serves a 64-bit access per half-warp (16 lanes x 8 bytes
must hit 16 distinct 8-byte slots of a 128-byte bank row) and a 128-bit access per quarter-warp (8
lanes x 16 bytes: 8 distinct 16-byte slots):

* the stage layout stage_byte(t, x, y) (k-term t, tile row x, column y) is a bijection onto the 4 KB
  of an operand, each producer cp.async instruction (one tile, 32 lanes x 16 bytes) fills 4 whole
  128-byte bank rows, and the DMMA fragment loads of every warp-tile mode (ragged or not) are
  conflict-free and sit at constant 512-byte steps per tile;
* the XOR-swizzled G-block gs(a,b,c,d) = Ta(a)^Tb(b)^Tc(c)^Td(d) is a bijection of [0,8)^4 onto
  [0,4096), every fold access is conflict-free per half-warp, and the epilogue's read conflicts are
  bounded.
"""
import itertools

Q, KB = 8, 8


def stage_byte(t, x, y):
    return 2048 * (t >> 2) + 512 * (x >> 1) + 128 * (t & 3) + 64 * (x & 1) + 16 * ((y >> 1) ^ (t & 3)) + 8 * (y & 1)


def test_stage_layout_bijection():
    assert sorted(stage_byte(t, x, y) for t in range(KB) for x in range(Q) for y in range(Q)) == \
        list(range(0, KB * 64 * 8, 8))


def test_producer_copies_fill_bank_rows():
    for kk in range(KB):
        for quarter in range(4):
            slots = set()
            rows = set()
            for lane in range(8 * quarter, 8 * quarter + 8):
                sr, sc2 = lane >> 2, lane & 3
                b = stage_byte(kk, sr, 2 * sc2)
                assert b % 16 == 0 and stage_byte(kk, sr, 2 * sc2 + 1) == b + 8
                rows.add(b // 128)
                slots.add((b % 128) // 16)
            assert len(rows) == 1 and len(slots) == 8, (kk, quarter)


def _tiles(MI, RY, wm):
    """(p, q) of the warp's M-tiles (csrc/schur.cu orient<>)."""
    qm, pm = (0, MI * wm) if RY else (wm, 0)
    return [(pm + i, qm) for i in range(MI)]


def test_fragment_loads_conflict_free_and_affine():
    for MI, RY in ((4, 0), (2, 0), (2, 1), (1, 1)):
        for wm in (0, 1):
            tiles = _tiles(MI, RY, wm)
            for k4 in (0, 1):
                base = None
                for i, (pp, qq) in enumerate(tiles):
                    for half in (0, 1):
                        slots = set()
                        for ln in range(16 * half, 16 * half + 16):
                            g, t = ln >> 2, ln & 3
                            x, y = 2 * pp + (g & 1), 4 * qq + (g >> 1)
                            assert x < Q and y < Q
                            b = stage_byte(t + 4 * k4, x, y)
                            slots.add((b % 128) // 8)
                            if i == 0 and half == 0 and ln == 0:
                                base = b
                        assert len(slots) == 16, (MI, RY, wm, k4, i, half)
                    # tile i of every lane at +512 i (one address register per operand)
                    for ln in range(32):
                        g, t = ln >> 2, ln & 3
                        b0 = stage_byte(t + 4 * k4, 2 * tiles[0][0] + (g & 1), 4 * tiles[0][1] + (g >> 1))
                        bi = stage_byte(t + 4 * k4, 2 * pp + (g & 1), 4 * qq + (g >> 1))
                        assert bi - b0 == 512 * i
            # the tiles of both warp rows cover the valid (x, y) rows exactly once
    for MI, RY, nx, ny in ((4, 0, 8, 8), (2, 0, 4, 8), (2, 1, 8, 4), (1, 1, 4, 4)):
        rows = [(2 * pp + (g & 1), 4 * qq + (g >> 1)) for wm in (0, 1) for pp, qq in _tiles(MI, RY, wm) for g in range(8)]
        assert sorted(rows) == sorted((x, y) for x in range(nx) for y in range(ny)), (MI, RY)


def _lin3(v, c0, c1, c2):
    return (c0 if v & 1 else 0) ^ (c1 if v & 2 else 0) ^ (c2 if v & 4 else 0)


def _Ta(a):
    return _lin3(a, 11, 3, 10)


def _Tb(b):
    return _lin3(b, 7, 21, 32)


def _Tc(c):
    return _lin3(c, 65, 135, 264)


def _Td(d):
    return _lin3(d, 525, 1027, 2048)


def test_gblock_swizzle_is_a_bijection():
    addrs = {_Ta(a) ^ _Tb(b) ^ _Tc(c) ^ _Td(d) for a, b, c, d in itertools.product(range(8), repeat=4)}
    assert addrs == set(range(4096))


def test_fold_accesses_conflict_free_per_half_warp():
    """Every fold store / load acc[i][j][e] -> Gs of every orientation (raw (x,y,z,w) -> (a,b,c,d) =
    o0 (w,x,y,z), o1 (w,x,z,y), o2 (x,w,y,z), o3 (x,w,z,y)), warp-tile mode and warp hits 16 distinct
    8-byte bank slots in each half-warp."""
    n = 0
    for (MI, RY), (NJ, RW) in itertools.product(((4, 0), (2, 0), (2, 1), (1, 1)), repeat=2):
        for o, warp in itertools.product(range(4), range(4)):
            wm, wn = warp >> 1, warp & 1
            mt, nt = _tiles(MI, RY, wm), _tiles(NJ, RW, wn)
            for (pp, qq), (pn, qn), e, half in itertools.product(mt, nt, range(2), range(2)):
                slots = []
                for ln in range(16 * half, 16 * half + 16):
                    g, t = ln >> 2, ln & 3
                    x, y = 2 * pp + (g & 1), 4 * qq + (g >> 1)
                    z, w = 2 * pn + e, 4 * qn + t
                    bx = (_Ta(x) if o & 2 else _Tb(x)) ^ (_Td(y) if o & 1 else _Tc(y))
                    bz = (_Tc(z) if o & 1 else _Td(z)) ^ (_Tb(w) if o & 2 else _Ta(w))
                    slots.append((bx ^ bz) % 16)
                assert len(set(slots)) == 16, (MI, RY, NJ, RW, o, warp, pp, qq, pn, qn, e, half)
                n += 1
    assert n > 0


def test_epilogue_read_conflicts_bounded():
    """The epilogue reads Gs with lanes along the diagonal-ordered (c, d) or (a, b) tables (the order
    that makes G stores contiguous): those sets are not subspaces, so a few half-warps take a second
    wavefront -- at most 22 extra slots over all table halves (v24's swizzle: 52 on the direct terms)."""
    diag = [(lc, lc + dlt) for dlt in range(-7, 8) for lc in range(max(0, -dlt), min(7, 7 - dlt) + 1)]
    extra = 0
    for valid, dg in ((diag, False), ([p for p in diag if p[0] <= p[1]], True)):
        for h0 in range(0, len(valid), 16):
            grp = valid[h0:h0 + 16]
            sets = [[(_Tc(c) ^ _Td(d)) % 16 for c, d in grp], [(_Ta(a) ^ _Tb(b)) % 16 for a, b in grp]]
            if dg:
                sets += [[(_Tc(d) ^ _Td(c)) % 16 for c, d in grp if c != d], [(_Ta(b) ^ _Tb(a)) % 16 for a, b in grp if a != b]]
            extra += sum(len(s) - len(set(s)) for s in sets)
    assert extra <= 22, extra

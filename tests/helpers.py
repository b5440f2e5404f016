"""Shared parity helpers: GPU store <-> oracle Blocks conversion and checks."""
import numpy as np

from oracle.oracle import Blocks

TOL = 1e-12  # north_star: values within 1e-12 relative (Frobenius), FP64


def to_store(ctx, b: Blocks):
    from paper_1910_13555_b200.store import LocalStore
    s = LocalStore(ctx, b.rsz, b.csz)
    if b.nblk:
        s.put_blocks(b.bi, b.bj, b.vals)
    return s


def from_store(s) -> Blocks:
    bi, bj, v = s.export()
    return Blocks(s.rsz.copy(), s.csz.copy(), bi, bj, v)


def frob(a, b):
    diff = float(np.sum((a - b) ** 2))
    ref = float(np.sum(b * b))
    return np.sqrt(diff) if ref == 0 else np.sqrt(diff / ref)


def assert_parity(got: Blocks, want: Blocks, tol=TOL, per_block=True):
    """Pattern bit-exact; values within tol (global and per-block Frobenius)."""
    assert got.nblk == want.nblk, f"block count {got.nblk} != {want.nblk}"
    assert np.array_equal(got.bi, want.bi) and np.array_equal(got.bj, want.bj), "pattern differs"
    assert got.vals.shape == want.vals.shape
    g = frob(got.vals, want.vals)
    assert g <= tol, f"global Frobenius rel err {g}"
    if per_block and want.nblk:
        off = want.offsets()[:-1]
        d = np.add.reduceat((got.vals - want.vals) ** 2, off)
        r = np.add.reduceat(want.vals ** 2, off)
        per = np.where(r == 0, np.sqrt(d), np.sqrt(d / np.where(r == 0, 1, r)))
        worst = float(per.max())
        assert worst <= tol, f"worst per-block Frobenius rel err {worst}"
    return g


def write_matrix_binary(path, b: Blocks):
    """The reference's binary matrix format (io.hpp:132-178), little endian."""
    import struct
    with open(path, "wb") as f:
        f.write(struct.pack("<4q", int(b.rsz.sum()), int(b.csz.sum()), len(b.rsz), len(b.csz)))
        f.write(np.asarray(b.rsz, "<i8").tobytes())
        f.write(np.asarray(b.csz, "<i8").tobytes())
        off = b.offsets()
        for t in range(b.nblk):
            f.write(struct.pack("<2q", int(b.bi[t]), int(b.bj[t])))
            f.write(np.asarray(b.vals[off[t]:off[t + 1]], "<f8").tobytes())


def read_matrix_binary(path) -> Blocks:
    raw = open(path, "rb").read()
    h = np.frombuffer(raw[:32], "<i8")
    nbr, nbc = int(h[2]), int(h[3])
    rsz = np.frombuffer(raw[32:32 + 8 * nbr], "<i8").astype(np.int32)
    csz = np.frombuffer(raw[32 + 8 * nbr:32 + 8 * (nbr + nbc)], "<i8").astype(np.int32)
    pos = 32 + 8 * (nbr + nbc)
    bi, bj, vals = [], [], []
    while pos < len(raw):
        i, j = np.frombuffer(raw[pos:pos + 16], "<i8")
        pos += 16
        n = int(rsz[i]) * int(csz[j])
        vals.append(np.frombuffer(raw[pos:pos + 8 * n], "<f8"))
        pos += 8 * n
        bi.append(i)
        bj.append(j)
    return Blocks(rsz, csz, np.array(bi, np.int64), np.array(bj, np.int64),
                  np.concatenate(vals) if vals else np.zeros(0))

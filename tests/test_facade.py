"""The C++ facade (include/blocktensor/b200.hpp): a caller written against the
reference API builds against it and reproduces the oracle through the C-ABI."""
import os
import subprocess

import numpy as np
import pytest

from helpers import assert_parity, read_matrix_binary, write_matrix_binary

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "multiply_files")


def _build():
    subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], check=True,
                   capture_output=True)


def test_facade_example_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
@pytest.mark.parametrize("algo,q,nprocs", [("cannon", 1, 1), ("cannon", 2, 4), ("case1", 1, 3),
                                           ("case2", 1, 4), ("auto", 2, 4), ("auto", 1, 2)])
def test_facade_multiply_matches_oracle(oracle, tmp_path, algo, q, nprocs):
    _build()
    rs = np.array([5, 13, 23, 7, 13, 5, 23, 11], np.int32)
    ks = np.array([13, 5, 23, 8, 16, 23], np.int32)
    ns = np.array([23, 7, 5, 13, 20], np.int32)
    A = oracle.random_matrix(21, rs, ks, 0.5)
    B = oracle.random_matrix(22, ks, ns, 0.5)
    Cin = oracle.random_matrix(23, rs, ns, 0.2)
    paths = [str(tmp_path / n) for n in ("a.bin", "b.bin", "c.bin", "out.bin")]
    for p, m in zip(paths, (A, B, Cin)):
        write_matrix_binary(p, m)
    r = subprocess.run([EXE, algo, str(q), str(nprocs)] + paths, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    want, _, _ = oracle.multiply(A, B, Cin)
    assert_parity(read_matrix_binary(paths[3]), want)


@pytest.mark.gpu
def test_facade_maps_errors(tmp_path, oracle):
    _build()
    A = oracle.random_matrix(1, [2, 2], [2, 2], 1.0)
    B = oracle.random_matrix(2, [3], [2], 1.0)  # nonconformal
    paths = [str(tmp_path / n) for n in ("a.bin", "b.bin", "c.bin", "out.bin")]
    write_matrix_binary(paths[0], A)
    write_matrix_binary(paths[1], B)
    write_matrix_binary(paths[2], A)
    r = subprocess.run([EXE, "cannon", "1", "1"] + paths, capture_output=True, text=True)
    assert r.returncode == 1 and "inner blockings" in r.stderr


def test_facade_tensor_example_compiles():
    _build()
    assert os.path.exists(os.path.join(ROOT, "examples", "contract_tensor"))


@pytest.mark.gpu
def test_facade_tensor_contraction():
    """C++ SparseTensor / contract through the C-ABI: the
    rank-3 (ab|P)(P|Q) contraction with a device remap of T, vs a dense host
    evaluation inside the example (exit 0 iff <= 1e-12)."""
    _build()
    r = subprocess.run([os.path.join(ROOT, "examples", "contract_tensor")], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "frobenius rel err" in r.stdout


def _special_values(oracle, seed=51):
    """a mixed-size matrix whose values include awkward doubles for the text
    format (signed zero, extremes of the normal range, non-terminating binary
    fractions)"""
    rs = np.array([3, 1, 4, 2], np.int32)
    cs = np.array([2, 5, 1], np.int32)
    m = oracle.random_matrix(seed, rs, cs, 0.7)
    v = m.vals.copy()
    special = [-0.0, 0.1, -1e-300, 2.2250738585072014e-308, 1.7976931348623157e308, 1 / 3, -7.0]
    v[:len(special)] = special[:len(v)]
    from oracle.oracle import Blocks
    return Blocks(m.rsz, m.csz, m.bi, m.bj, v)


@pytest.mark.gpu
@pytest.mark.parametrize("fin,fout", [("binary", "binary"), ("text", "text"), ("text", "binary"),
                                      ("binary", "text")])
def test_facade_io_matches_reference_io(reference, oracle, tmp_path, fin, fout):
    """Fixture I/O pinned to the reference's own io.hpp (compiled, unmodified):
    the facade reads what the reference wrote and writes byte-identical files;
    the reference reads the facade's files back to the same blocks."""
    _build()
    m = _special_values(oracle)
    src, ref_out, ours = (str(tmp_path / n) for n in ("src", "ref_out", "ours"))
    reference.write_matrix_file(src, m, fin)
    reference.write_matrix_file(ref_out, m, fout)
    r = subprocess.run([os.path.join(ROOT, "examples", "convert_matrix"), src, fin, ours, fout],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert open(ours, "rb").read() == open(ref_out, "rb").read()
    back = reference.read_matrix_file(ours, fout)
    assert np.array_equal(back.bi, m.bi) and np.array_equal(back.bj, m.bj)
    assert np.array_equal(back.vals.view(np.int64), m.vals.view(np.int64))   # bit-exact


@pytest.mark.gpu
def test_facade_api_surface():
    """Axis::functional, LocalStore::for_each, put/get_block_at ownership,
    for_each_global, redistribute (transpose) / redistribute_add + ledger."""
    _build()
    r = subprocess.run([os.path.join(ROOT, "examples", "facade_api")], capture_output=True,
                       text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("OK:") >= 8 and "FAIL" not in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("world,algo,q,nprocs", [(4, "cannon", 2, 4), (2, "case2", 1, 2),
                                                 (2, "case1", 1, 2)])
def test_facade_multiply_files_nccl(oracle, tmp_path, world, algo, q, nprocs):
    """examples/multiply_files under torchrun: one rank per GPU over NCCL through
    the facade's SimComm(grid, device, rank, NcclId), each rank writing its C
    blocks; the union equals the oracle."""
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import sys
    _build()
    rs = np.array([5, 13, 23, 7, 13, 5, 23, 11], np.int32)
    ks = np.array([13, 5, 23, 8, 16, 23], np.int32)
    ns = np.array([23, 7, 5, 13, 20], np.int32)
    A = oracle.random_matrix(61, rs, ks, 0.5)
    B = oracle.random_matrix(62, ks, ns, 0.5)
    Cin = oracle.random_matrix(63, rs, ns, 0.2)
    paths = [str(tmp_path / n) for n in ("a.bin", "b.bin", "c.bin", "out.bin")]
    for p, m in zip(paths, (A, B, Cin)):
        write_matrix_binary(p, m)
    port = 29700 + world + (0 if algo == "cannon" else 7 if algo == "case2" else 13)
    env = dict(os.environ, BT_NCCL_ID_FILE=str(tmp_path / "nccl_id"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           "--no-python", EXE, algo, str(q), str(nprocs)] + paths
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    parts = [read_matrix_binary(paths[3] + f".rank{k}") for k in range(world)]
    from oracle.oracle import Blocks
    bi = np.concatenate([p.bi for p in parts])
    bj = np.concatenate([p.bj for p in parts])
    blocks = []
    for p in parts:
        off = p.offsets()
        blocks += [p.vals[off[t]:off[t + 1]] for t in range(p.nblk)]
    order = np.lexsort((bj, bi))
    got = Blocks(rs, ns, bi[order], bj[order], np.concatenate([blocks[t] for t in order]))
    want, _, _ = oracle.multiply(A, B, Cin)
    assert_parity(got, want)


def _ts_case(oracle, tmp_path):
    rs = np.array([4, 3, 5, 4, 2, 4, 3, 5], np.int32)        # M: 8 blocks
    ks = np.array([3, 4, 5, 2] * 32, np.int32)               # K: 128 blocks (the long dim)
    ns = np.array([5, 4, 3, 4, 4, 2, 5, 3], np.int32)        # N: 8 blocks
    A = oracle.random_matrix(81, rs, ks, 0.5)
    B = oracle.random_matrix(82, ks, ns, 0.5)
    pa, pb, pc = (str(tmp_path / n) for n in ("a.bin", "b.bin", "c.bin"))
    write_matrix_binary(pa, A)
    write_matrix_binary(pb, B)
    from oracle.oracle import Blocks
    want, _, _ = oracle.multiply(A, B, Blocks.empty(rs, ns))
    return (rs, ns), pa, pb, pc, want


def _merge_parts(paths, rs, ns):
    from oracle.oracle import Blocks
    parts = [read_matrix_binary(p) for p in paths]
    bi = np.concatenate([p.bi for p in parts])
    bj = np.concatenate([p.bj for p in parts])
    blocks = []
    for p in parts:
        off = p.offsets()
        blocks += [p.vals[off[t]:off[t + 1]] for t in range(p.nblk)]
    order = np.lexsort((bj, bi))
    vals = np.concatenate([blocks[t] for t in order]) if len(order) else np.zeros(0)
    return Blocks(rs, ns, bi[order], bj[order], vals)


@pytest.mark.gpu
@pytest.mark.parametrize("f,sr,sc", [(1, 2, 2), (2, 2, 1), (4, 1, 1)])
def test_facade_tall_skinny_virtual_subgroups(oracle, tmp_path, f, sr, sc):
    """C++ tall-skinny layer, K split into f subgroups of
    virtual ranks (SPEC example: A 8x128 blocks split f=4 on K, B 128x8):
    C equals the oracle; the cross-subgroup reduction is charged to the
    ledger (f > 1); a 10^4-block split dimension keeps no host index array and
    device index ranges of one submatrix (ceil(10^4/f))."""
    _build()
    (rs, ns), pa, pb, pc, want = _ts_case(oracle, tmp_path)
    r = subprocess.run([os.path.join(ROOT, "examples", "tall_skinny"), str(f), str(sr), str(sc),
                        pa, pb, pc], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert_parity(_merge_parts([pc], rs, ns), want)
    import re
    m = re.search(r"ts_reduce elements sent (\d+), host index entries (\d+), max device index "
                  r"range (\d+)", r.stdout)
    assert m, r.stdout
    assert (int(m.group(1)) > 0) == (f > 1)
    assert int(m.group(2)) == 0 and int(m.group(3)) == -(-10000 // f)


@pytest.mark.gpu
@pytest.mark.parametrize("f,sr,sc", [(2, 2, 1), (4, 1, 1)])
def test_facade_tall_skinny_nccl_subgroups(oracle, tmp_path, f, sr, sc):
    """The same with one rank per GPU: subgroups are NCCL communicators split
    from the parent (bt_ctx_split) and multiply concurrently."""
    import sys
    import torch
    world = f * sr * sc
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    _build()
    (rs, ns), pa, pb, pc, want = _ts_case(oracle, tmp_path)
    env = dict(os.environ, BT_NCCL_ID_FILE=str(tmp_path / "nccl_id"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(29750 + f), "--no-python", os.path.join(ROOT, "examples", "tall_skinny"),
           str(f), str(sr), str(sc), pa, pb, pc]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert_parity(_merge_parts([pc + f".rank{k}" for k in range(world)], rs, ns), want)

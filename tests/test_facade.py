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
                                           ("case2", 1, 4)])
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

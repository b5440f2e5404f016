"""BASELINE config 4 through the tensor API: R_(ab)Q += sum_P T_(ab)P M_PQ with
contract(), on one GPU.

  python tools/run_c4_contract.py [--steps K]

The inputs are tools/run_config.py's c4 (a, b: 200 AO blocks, P, Q: 400 aux
blocks, sizes 13/23 alternating, T occupancy 0.001, (P|Q) band 7).  T is a
rank-3 SparseTensor (a, b, P); its matricization ((a,b),(P)) with b fastest is
exactly run_config's matrix, so the values go in as they are.  Two timings:

  compatible  T in ((a,b),(P)), M in ((P),(Q)), R in ((a,b),(Q)): contract()
              multiplies directly (no remap, SPEC.md "fast path");
  remapped    T stored as ((a),(b,P)): contract() first remaps it on the
              device into ((a,b),(P)) (bt_tensor_remap), then multiplies.

CUDA events on the context stream around each contract() call, L2 flushed.
Parity of this contraction at full size (both layouts, against the oracle):
tests/test_configs_gpu.py::test_c4_through_contract_full_size.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch
    from run_config import config
    from paper_1910_13555_b200.store import Context
    from paper_1910_13555_b200.tensor import SparseTensor, contract
    rng = np.random.default_rng(2024)
    rows, aux, _, T, M, eps, desc = config("c4", rng)
    ao = np.tile(np.array([13, 23], np.int32), 100)
    ctx = Context(0)
    ctx.set_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t = SparseTensor(ctx, [ao, ao, aux], [0, 1], [2])
    t.store.put_blocks(*T)
    m = SparseTensor(ctx, [aux, aux], [0], [1])
    m.store.put_blocks(*M)
    t_alt = t.remap([0], [1, 2])       # the same tensor stored as ((a),(b,P))
    out = {"config": "c4 via contract()", "workload": desc}

    def timed(fn):
        ms = []
        for it in range(2 + args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            st = fn()
            with torch.cuda.stream(stream):
                e1.record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                ms.append(e0.elapsed_time(e1))
        return float(np.median(ms)), st

    r = SparseTensor(ctx, [ao, ao, aux], [0, 1], [2])

    def contract_into(src):
        r.store.clear()   # R's slab is kept as capacity (no 11 GB allocation per call)
        return contract(src, m, [2], [0], r)

    ms_c, st = timed(lambda: contract_into(t))
    ms_r, _ = timed(lambda: contract_into(t_alt))
    t_back = SparseTensor(ctx, [ao, ao, aux], [0, 1], [2])
    ms_remap, _ = timed(lambda: t_alt.remap_into_store(t_back))
    out.update({"products": st["products"], "useful_gflop": round(st["flops"] / 1e9, 3),
                "compatible_ms": round(ms_c, 4), "remapped_ms": round(ms_r, 4),
                "remap_only_ms": round(ms_remap, 4),
                "remap_share_of_multiply": round(ms_remap / ms_c, 4),
                "compatible_tflops": round(st["flops"] / ms_c / 1e9, 3),
                "remapped_tflops": round(st["flops"] / ms_r / 1e9, 3),
                "t_elements": int(t.store.info()[1])})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

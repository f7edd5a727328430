"""Generate tests/golden/golden.npz from the REFERENCE ITSELF.

Runs in the build container (needs oracle/_ref/libccsim_ref.so, compiled from
/root/reference by `make -C oracle ref`). Every vector below is produced by the
reference's own code — ccsim::NvrarAllreduce<T>::run on the virtual-time engine,
oracles::random_inputs, oracles::nvrar_order_sum — never by this repo's
restatement, so the fixtures pin the restatement (tests/test_oracle.py) and,
through it, the GPU path (tests/test_gpu_parity.py).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
META = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_meta.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    assert O.ref_available(), "build oracle/_ref first: make -C oracle ref"
    g: dict[str, np.ndarray] = {}
    meta: dict[str, object] = {}

    # 1. the input generator (tests/oracles.hpp:161-178)
    g["rand_f32_8x64_s1234"] = O.ref_random_inputs(8, 64, 1234, "f32")
    g["rand_i32_4x64_s13"] = O.ref_random_inputs(4, 64, 13, "i32")

    # 2. NvrarAllreduce<float>::run per hierarchy, n = 1031 (padding), seed 19.
    #    All ranks must agree; one row is stored per hierarchy.
    hiers = [(1, 1), (1, 2), (2, 1), (1, 4), (2, 2), (4, 1), (1, 8), (2, 4), (4, 2), (8, 1),
             (2, 3), (4, 3), (8, 2), (8, 4)]
    for nodes, gpus in hiers:
        p = nodes * gpus
        x = O.ref_random_inputs(p, 1031, 19, "f32")
        out = O.ref_nvrar_run_all(x, nodes, gpus, blocks=2, chunk_bytes=64)
        assert all(np.array_equal(out[0].view(np.uint32), out[r].view(np.uint32))
                   for r in range(p))
        g[f"nvrar_f32_{nodes}x{gpus}_n1031_s19"] = out[0]

    # 3. collectives_test.cpp:379-390 — float32, 4x2, n=129, seed 19
    x = O.ref_random_inputs(8, 129, 19, "f32")
    g["ct_float_4x2_n129_s19"] = O.ref_nvrar_run_all(x, 4, 2)[0]
    # collectives_test.cpp:372-378 — int32, 4x4, n=999, seed 13
    x = O.ref_random_inputs(16, 999, 13, "i32")
    g["ct_int_4x4_n999_s13"] = O.ref_nvrar_run_all(x, 4, 4)[0]
    # collectives_test.cpp:364-371 — 2x2, inputs {g} -> {6}
    g["ct_2x2_pad"] = O.ref_nvrar_run_all(np.arange(4, dtype=np.int32).reshape(4, 1), 2, 2)[0]

    # 4. SURVEY §8c: 2x4, 1 MB fp32, seed 1234 (C1) — too big to store; hash of the bits.
    x = O.ref_random_inputs(8, 262144, 1234, "f32")
    out = O.ref_nvrar_run_all(x, 2, 4, blocks=8, chunk_bytes=16384)
    meta["c1_2x4_1MB_f32_s1234_sha256"] = sha(out[0])
    meta["c1_differs_from_serial"] = int(np.count_nonzero(
        out[0].view(np.uint32) != O.serial_sum(x).view(np.uint32)))
    # bf16 rule: fp32 reference on up-cast bf16 inputs, rounded once.
    xb = O.bf16_bits_from_f32(x)
    outb = O.ref_nvrar_run_all(O.f32_from_bf16_bits(xb).reshape(8, -1), 2, 4)
    meta["c2_2x4_1MB_bf16_s1234_sha256"] = sha(O.bf16_bits_from_f32(outb[0]))

    # 5. acceptance criterion 1 (acceptance_test.cpp:85-112), int32 == serial: hashes.
    acc = {}
    seed = 100
    for n in (1, 2, 4, 8):
        for gp in (1, 2, 4):
            for nbytes in (8, 1024, 65536, 131072, 1048576):
                seed += 1
                elems = nbytes // 4
                x = O.ref_random_inputs(n * gp, elems, seed, "i32")
                out = O.ref_nvrar_run_all(x, n, gp)
                assert all(np.array_equal(out[0], out[r]) for r in range(n * gp))
                acc[f"{n}x{gp}_{nbytes}_s{seed}"] = sha(out[0])
    meta["acceptance1_sha256"] = acc

    # 6. stalled rank (collectives_test.cpp:462-497): blocked set rows.
    rc, rows, msg = O.ref_stalled_rank(4, 1, 32, 3, 31, 32)
    assert rc == 5
    g["stalled_4x1_rows"] = rows
    meta["stalled_4x1_msg"] = msg

    # 7. standalone phases (collectives_test.cpp:179-354): IntraReduceScatter /
    # IntraAllGather with each node's members, NvrarAllreduce::rd_inter.
    g["rs_i32_1x2_hand"] = O.ref_intra_phase("rs", np.array([[1, 2], [3, 4]], np.int32), 1, 2)
    for nodes, gpus, n, dt, seed in [(1, 4, 64, "i32", 17), (2, 4, 1031, "f32", 19),
                                     (1, 3, 1000, "f32", 21), (2, 3, 4099, "f32", 23)]:
        x = O.ref_random_inputs(nodes * gpus, n, seed, dt)
        rs = O.ref_intra_phase("rs", x, nodes, gpus)
        g[f"rs_{dt}_{nodes}x{gpus}_n{n}_s{seed}"] = rs
        ag = O.ref_intra_phase("ag", rs, nodes, gpus)
        meta[f"ag_{dt}_{nodes}x{gpus}_n{n}_s{seed}_sha256"] = sha(ag)
    for nodes, gpus, w, dt, seed in [(8, 2, 96, "i32", 5), (4, 2, 777, "f32", 29),
                                     (8, 1, 1000, "f32", 31), (2, 4, 100, "f32", 37)]:
        x = O.ref_random_inputs(nodes * gpus, w, seed, dt)
        g[f"rd_{dt}_{nodes}x{gpus}_w{w}_s{seed}"] = O.ref_rd_inter(x, nodes, gpus)

    # 8. the reference's baseline collectives: RingAllreduce / TreeAllreduce
    # result bits (ring.hpp, tree.hpp) per hierarchy, n = 1031, seed 19.
    bl = {}
    for nodes, gpus in [(1, 2), (2, 1), (1, 4), (2, 2), (4, 1), (1, 8), (2, 4), (4, 2), (8, 1),
                        (2, 3), (8, 2)]:
        x = O.ref_random_inputs(nodes * gpus, 1031, 19, "f32")
        for which in ("ring", "tree"):
            out = O.ref_baseline_run_all(which, x, nodes, gpus)
            assert all(np.array_equal(out[0], out[r]) for r in range(nodes * gpus))
            bl[f"{which}_{nodes}x{gpus}"] = sha(out[0])
    g["ring_f32_2x4_n1031_s19"] = O.ref_baseline_run_all(
        "ring", O.ref_random_inputs(8, 1031, 19, "f32"), 2, 4)[0]
    g["tree_f32_2x4_n1031_s19"] = O.ref_baseline_run_all(
        "tree", O.ref_random_inputs(8, 1031, 19, "f32"), 2, 4)[0]
    meta["baseline_orders_n1031_s19_sha256"] = bl

    np.savez_compressed(OUT, **g)
    with open(META, "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} B) and {META}")


if __name__ == "__main__":
    main()

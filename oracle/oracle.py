"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front-end of the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline
leg and ``--impl reference`` arm) may import this module, and only as the
checker / the timed CPU baseline. The product package never imports it.

Two libraries sit behind it:

* ``oracle/liboracle_nvrar.so`` — the plain-C restatement (``nvrar_oracle.c``)
  of the reference's arithmetic: ``oracles::random_inputs``
  (tests/oracles.hpp:161-178), ``oracles::nvrar_order_sum``
  (tests/oracles.hpp:101-133), ``serial_sum`` (:25-34), fused words
  (transport.hpp:81-87).
* ``oracle/_ref/libccsim_ref.so`` — the reference's own headers compiled
  unmodified (``oracle/ref_shim.cpp``): ``ccsim::NvrarAllreduce<T>`` on the
  virtual-time and concurrent engines. Optional: present when it was built in
  the container that had /root/reference (it travels to the GPU box prebuilt).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_nvrar.so")
REF_PATH = os.path.join(HERE, "_ref", "libccsim_ref.so")

INT32, FLOAT32, BF16 = 0, 1, 2

_lib = None
_ref = None


def build(ref: bool = True) -> None:
    """Compile the C restatement (and the reference shim when /root/reference exists)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    if ref and os.path.isdir("/root/reference/proj/include"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = ctypes.CDLL(LIB_PATH)
        c_sz, c_u64, vp = ctypes.c_size_t, ctypes.c_uint64, ctypes.c_void_p
        L.orc_random_inputs_f32.argtypes = [ctypes.c_int, c_sz, c_u64, vp]
        L.orc_random_inputs_i32.argtypes = [ctypes.c_int, c_sz, c_u64, vp]
        for name in ("orc_nvrar_order_sum_f32", "orc_nvrar_order_sum_i32",
                     "orc_nvrar_order_sum_bf16"):
            getattr(L, name).argtypes = [ctypes.c_int, ctypes.c_int, c_sz, vp, vp]
            getattr(L, name).restype = ctypes.c_int
        for name in ("orc_ring_order_sum_f32", "orc_ring_order_sum_i32",
                     "orc_tree_order_sum_f32", "orc_tree_order_sum_i32"):
            getattr(L, name).argtypes = [ctypes.c_int, ctypes.c_int, c_sz, vp, vp]
            getattr(L, name).restype = ctypes.c_int
        for name in ("orc_intra_rs_sum_f32", "orc_intra_rs_sum_i32"):
            getattr(L, name).argtypes = [ctypes.c_int, c_sz, vp, vp]
            getattr(L, name).restype = ctypes.c_int
        for name in ("orc_rd_inter_f32", "orc_rd_inter_i32"):
            getattr(L, name).argtypes = [ctypes.c_int, ctypes.c_int, c_sz, vp, vp]
            getattr(L, name).restype = ctypes.c_int
        L.orc_serial_sum_f32.argtypes = [ctypes.c_int, c_sz, vp, vp]
        L.orc_serial_sum_i32.argtypes = [ctypes.c_int, c_sz, vp, vp]
        L.orc_make_word.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.orc_make_word.restype = c_u64
        L.orc_unpack_fused.argtypes = [vp, c_sz, ctypes.c_uint32, vp, ctypes.POINTER(c_sz)]
        L.orc_unpack_fused.restype = ctypes.c_int
        L.orc_pack_fused.argtypes = [vp, c_sz, ctypes.c_uint32, vp]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_PATH} not built (needs /root/reference)")
        R = ctypes.CDLL(REF_PATH)
        c_sz, c_u64, vp, ci, cd = (ctypes.c_size_t, ctypes.c_uint64, ctypes.c_void_p,
                                   ctypes.c_int, ctypes.c_double)
        R.ref_random_inputs_f32.argtypes = [ci, c_sz, c_u64, vp]
        R.ref_random_inputs_i32.argtypes = [ci, c_sz, c_u64, vp]
        R.ref_nvrar_order_sum_f32.argtypes = [ci, ci, c_sz, vp, vp]
        R.ref_nvrar_order_sum_i32.argtypes = [ci, ci, c_sz, vp, vp]
        R.ref_serial_sum_f32.argtypes = [ci, c_sz, vp, vp]
        for name in ("ref_nvrar_run_all_f32", "ref_nvrar_run_all_i32"):
            getattr(R, name).argtypes = [ci, ci, c_sz, vp, vp, ci, c_u64, ci, c_u64, cd, cd,
                                         ctypes.c_char_p, c_sz]
            getattr(R, name).restype = ci
        R.ref_nvrar_time_concurrent_f32.argtypes = [ci, ci, c_sz, vp, ci, c_u64, ci, ci, vp,
                                                    ctypes.c_char_p, c_sz]
        R.ref_nvrar_time_concurrent_f32.restype = ci
        R.ref_nvrar_stalled_rank.argtypes = [ci, ci, c_sz, ci, c_u64, c_u64, vp, ci,
                                             ctypes.POINTER(ci), ctypes.c_char_p, c_sz]
        R.ref_nvrar_stalled_rank.restype = ci
        for name in ("ref_intra_rs_f32", "ref_intra_rs_i32", "ref_intra_ag_f32",
                     "ref_intra_ag_i32"):
            getattr(R, name).argtypes = [ci, ci, c_sz, vp, vp, ctypes.c_char_p, c_sz]
            getattr(R, name).restype = ci
        for name in ("ref_ring_run_all_f32", "ref_ring_run_all_i32", "ref_tree_run_all_f32",
                     "ref_tree_run_all_i32"):
            getattr(R, name).argtypes = [ci, ci, c_sz, vp, vp, ctypes.c_char_p, c_sz]
            getattr(R, name).restype = ci
        for name in ("ref_rd_inter_f32", "ref_rd_inter_i32"):
            getattr(R, name).argtypes = [ci, ci, c_sz, vp, vp, ci, c_u64, ctypes.c_char_p, c_sz]
            getattr(R, name).restype = ci
        _ref = R
    return _ref


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# ---- restatement ---------------------------------------------------------

def random_inputs(ranks: int, n: int, seed: int, dtype: str = "f32") -> np.ndarray:
    """oracles::random_inputs<T> (tests/oracles.hpp:161-178) -> [ranks, n]."""
    if dtype == "f32":
        out = np.empty((ranks, n), np.float32)
        lib().orc_random_inputs_f32(ranks, n, seed, _ptr(out))
    elif dtype == "i32":
        out = np.empty((ranks, n), np.int32)
        lib().orc_random_inputs_i32(ranks, n, seed, _ptr(out))
    else:
        raise ValueError(dtype)
    return out


def bf16_bits_from_f32(x: np.ndarray) -> np.ndarray:
    """RNE fp32 -> bf16, returned as uint16 bits (NaN quieted)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    nan = ((u & 0x7F800000) == 0x7F800000) & ((u & 0x007FFFFF) != 0)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def f32_from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


def nvrar_order_sum(inputs: np.ndarray, nodes: int, gpus: int, dtype: str = "f32") -> np.ndarray:
    """Reference reduction order for hierarchy nodes x gpus (oracles.hpp:101-133).

    inputs: [nodes*gpus, n] (float32, int32, or uint16 bf16 bits for dtype='bf16').
    """
    inputs = np.ascontiguousarray(inputs)
    p, n = inputs.shape
    assert p == nodes * gpus
    fn = {"f32": ("orc_nvrar_order_sum_f32", np.float32),
          "i32": ("orc_nvrar_order_sum_i32", np.int32),
          "bf16": ("orc_nvrar_order_sum_bf16", np.uint16)}[dtype]
    inputs = inputs.astype(fn[1], copy=False)
    out = np.empty(n, fn[1])
    rc = getattr(lib(), fn[0])(nodes, gpus, n, _ptr(inputs), _ptr(out))
    if rc == -1:
        raise ValueError(f"nodes={nodes} is not a power of two")
    if rc != 0:
        raise RuntimeError(f"oracle rc={rc}")
    return out


def order_sum(inputs: np.ndarray, nodes: int, gpus: int, order: str = "nvrar",
              dtype: str = "f32") -> np.ndarray:
    """The result bits of the reference's three all-reduces for hierarchy
    nodes x gpus: 'nvrar' (oracles.hpp:101-133), 'ring' (ring_order_sum,
    :67-86), 'tree' (tree_order_sum, :137-159). bf16 = the fp32 order sum of
    the up-cast inputs, one RNE rounding."""
    if order == "nvrar":
        return nvrar_order_sum(inputs, nodes, gpus, dtype)
    x = np.ascontiguousarray(inputs)
    if dtype == "bf16":
        return bf16_bits_from_f32(order_sum(f32_from_bf16_bits(x), nodes, gpus, order, "f32"))
    p, n = x.shape
    assert p == nodes * gpus
    suffix = "f32" if dtype == "f32" else "i32"
    x = x.astype(np.float32 if suffix == "f32" else np.int32, copy=False)
    out = np.empty(n, x.dtype)
    rc = getattr(lib(), f"orc_{order}_order_sum_{suffix}")(nodes, gpus, n, _ptr(x), _ptr(out))
    if rc == -1:
        raise ValueError(f"nodes={nodes} is not a power of two")
    if rc != 0:
        raise RuntimeError(f"oracle rc={rc}")
    return out


def intra_rs_sum(node_inputs: np.ndarray) -> np.ndarray:
    """tests/oracles.hpp:89-97: the node-local ring reduce-scatter result,
    zero-padded to ceil(n/G)*G elements (chunk g = local rank g's shard)."""
    x = np.ascontiguousarray(node_inputs)
    g, n = x.shape
    name = {np.dtype(np.float32): "orc_intra_rs_sum_f32", np.dtype(np.int32): "orc_intra_rs_sum_i32"}[x.dtype]
    out = np.empty(-(-n // g) * g, x.dtype)
    if getattr(lib(), name)(g, n, _ptr(x), _ptr(out)) != 0:
        raise RuntimeError("oracle intra_rs_sum failed")
    return out


def rd_inter(shards: np.ndarray, nodes: int, gpus: int) -> np.ndarray:
    """NvrarAllreduce::rd_inter result (nvrar.hpp:132-155): per local rank, the
    XOR-step sum of its node peers' shards. shards: [P, w] -> [P, w]."""
    x = np.ascontiguousarray(shards)
    p, w = x.shape
    assert p == nodes * gpus
    name = {np.dtype(np.float32): "orc_rd_inter_f32", np.dtype(np.int32): "orc_rd_inter_i32"}[x.dtype]
    out = np.empty_like(x)
    rc = getattr(lib(), name)(nodes, gpus, w, _ptr(x), _ptr(out))
    if rc == -1:
        raise ValueError(f"nodes={nodes} is not a power of two")
    if rc != 0:
        raise RuntimeError(f"oracle rc={rc}")
    return out


def pack_fused(data_bits: np.ndarray, seq: int) -> np.ndarray:
    """fused.hpp pack: word = data (low 32 bits) | seq << 32 (transport.hpp:81-87)."""
    d = np.ascontiguousarray(data_bits).view(np.uint32).astype(np.uint64)
    return d | (np.uint64(seq) << np.uint64(32))


def unpack_fused(words: np.ndarray, seq: int, dtype=np.int32) -> np.ndarray:
    """fused.hpp unpack: every flag must equal seq (else the reference throws)."""
    w = np.ascontiguousarray(words).astype(np.uint64)
    flags = (w >> np.uint64(32)).astype(np.uint32)
    if np.any(flags != np.uint32(seq)):
        raise ValueError("stale flag")
    return (w & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(dtype)


def serial_sum(inputs: np.ndarray) -> np.ndarray:
    inputs = np.ascontiguousarray(inputs)
    p, n = inputs.shape
    out = np.empty(n, inputs.dtype)
    if inputs.dtype == np.float32:
        lib().orc_serial_sum_f32(p, n, _ptr(inputs), _ptr(out))
    elif inputs.dtype == np.int32:
        lib().orc_serial_sum_i32(p, n, _ptr(inputs), _ptr(out))
    else:
        raise ValueError(inputs.dtype)
    return out


def nvrar_order_sum_numpy(inputs: np.ndarray, nodes: int, gpus: int) -> np.ndarray:
    """Vectorised numpy restatement of the same order (float32 / int32 only).

    numpy's elementwise float32 add rounds each operation exactly like the C
    restatement; int32 adds wrap. Used to cross-check the C oracle at sizes
    where a scalar loop would be slow.
    """
    p, n = inputs.shape
    shard = -(-n // gpus)
    x = inputs.reshape(nodes, gpus, n)
    e = np.arange(n)
    c = e // shard
    v = []
    with np.errstate(over="ignore"):
        for node in range(nodes):
            xs = x[node]
            if gpus == 1:
                f = xs[0].copy()
            else:
                f = xs[(c + 1) % gpus, e].copy()
                for j in range(2, gpus):
                    f = f + xs[(c + j) % gpus, e]
                f = f + xs[c, e]
            v.append(f)
        bit = 1
        while bit < nodes:
            v = [v[node ^ bit] + v[node] for node in range(nodes)]
            bit <<= 1
    return v[0]


# ---- the reference itself -----------------------------------------------

class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def ref_random_inputs(ranks: int, n: int, seed: int, dtype: str = "f32") -> np.ndarray:
    if dtype == "f32":
        out = np.empty((ranks, n), np.float32)
        ref().ref_random_inputs_f32(ranks, n, seed, _ptr(out))
    else:
        out = np.empty((ranks, n), np.int32)
        ref().ref_random_inputs_i32(ranks, n, seed, _ptr(out))
    return out


def ref_order_sum(inputs: np.ndarray, nodes: int, gpus: int) -> np.ndarray:
    inputs = np.ascontiguousarray(inputs)
    out = np.empty(inputs.shape[1], inputs.dtype)
    fn = ref().ref_nvrar_order_sum_f32 if inputs.dtype == np.float32 else \
        ref().ref_nvrar_order_sum_i32
    fn(nodes, gpus, inputs.shape[1], _ptr(inputs), _ptr(out))
    return out


def ref_nvrar_run_all(inputs: np.ndarray, nodes: int, gpus: int, blocks: int = 1,
                      chunk_bytes: int = 65536, concurrent: bool = False, seed: int = 0,
                      delay_us: float = 0.0, timeout_s: float = 20.0) -> np.ndarray:
    """Run ccsim::NvrarAllreduce<T>::run on every rank; returns [P, n] outputs."""
    inputs = np.ascontiguousarray(inputs)
    out = np.empty_like(inputs)
    err = ctypes.create_string_buffer(512)
    fn = ref().ref_nvrar_run_all_f32 if inputs.dtype == np.float32 else \
        ref().ref_nvrar_run_all_i32
    rc = fn(nodes, gpus, inputs.shape[1], _ptr(inputs), _ptr(out), blocks, chunk_bytes,
            1 if concurrent else 0, seed, delay_us, timeout_s, err, 512)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return out


def ref_intra_phase(which: str, inputs: np.ndarray, nodes: int, gpus: int) -> np.ndarray:
    """Every rank runs ccsim::IntraReduceScatter<T> ('rs': [P, n] -> [P, ceil(n/G)])
    or IntraAllGather<T> ('ag': [P, ce] -> [P, G*ce]) with its node's members."""
    x = np.ascontiguousarray(inputs)
    p, ln = x.shape
    out_len = -(-ln // gpus) if which == "rs" else ln * gpus
    out = np.empty((p, out_len), x.dtype)
    suffix = "f32" if x.dtype == np.float32 else "i32"
    err = ctypes.create_string_buffer(512)
    rc = getattr(ref(), f"ref_intra_{which}_{suffix}")(nodes, gpus, ln, _ptr(x), _ptr(out), err, 512)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return out


def ref_baseline_run_all(which: str, inputs: np.ndarray, nodes: int, gpus: int) -> np.ndarray:
    """Every rank runs ccsim::RingAllreduce<T> ('ring') or TreeAllreduce<T> ('tree')."""
    x = np.ascontiguousarray(inputs)
    out = np.empty_like(x)
    suffix = "f32" if x.dtype == np.float32 else "i32"
    err = ctypes.create_string_buffer(512)
    rc = getattr(ref(), f"ref_{which}_run_all_{suffix}")(nodes, gpus, x.shape[1], _ptr(x),
                                                          _ptr(out), err, 512)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return out


def ref_rd_inter(shards: np.ndarray, nodes: int, gpus: int, blocks: int = 1,
                 chunk_bytes: int = 65536) -> np.ndarray:
    """Every rank runs ccsim::NvrarAllreduce<T>::rd_inter on its fused-packed shard
    (the collectives_test.cpp:286-302 driver); returns the unpacked [P, w] results."""
    x = np.ascontiguousarray(shards)
    out = np.empty_like(x)
    suffix = "f32" if x.dtype == np.float32 else "i32"
    err = ctypes.create_string_buffer(512)
    rc = getattr(ref(), f"ref_rd_inter_{suffix}")(nodes, gpus, x.shape[1], _ptr(x), _ptr(out),
                                                   blocks, chunk_bytes, err, 512)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return out


def ref_time_concurrent(inputs: np.ndarray, nodes: int, gpus: int, blocks: int = 1,
                        chunk_bytes: int = 65536, warmup: int = 2, calls: int = 10) -> np.ndarray:
    """Per-call makespan deltas (µs) of NvrarAllreduce<float> on ConcurrentEngine."""
    inputs = np.ascontiguousarray(inputs, np.float32)
    per = np.empty(calls, np.float64)
    err = ctypes.create_string_buffer(512)
    rc = ref().ref_nvrar_time_concurrent_f32(nodes, gpus, inputs.shape[1], _ptr(inputs), blocks,
                                             chunk_bytes, warmup, calls, _ptr(per), err, 512)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return per


def ref_stalled_rank(nodes: int, gpus: int, n: int, stall_rank: int, seed1: int, seed2: int):
    """Blocked set of the reference's stalled-rank fixture (collectives_test.cpp:462-497).

    Returns (rc, rows[k, 4] = {rank, kind 0=FlagWait/1=SeqWait, peer, expected}, message).
    Runs oracle/_ref/ref_tool in a subprocess (see ref_shim.cpp for why).
    """
    tool = os.path.join(HERE, "_ref", "ref_tool")
    out = subprocess.run([tool, "stalled", str(nodes), str(gpus), str(n), str(stall_rank),
                          str(seed1), str(seed2)], capture_output=True, text=True,
                         check=True).stdout.splitlines()
    rc = int(out[0].split()[1])
    rows = [list(map(int, ln.split())) for ln in out[1:] if not ln.startswith("msg")]
    msg = [ln for ln in out if ln.startswith("msg")][0][4:]
    return rc, np.array(rows, np.int32).reshape(-1, 4), msg

"""Thin ctypes binding of include/slc.h (libslc.so) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module converts torch tensors / Python values to pointers and sizes and
raises on a non-OK status.  There is no fallback: if libslc.so is missing the
import-time load fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLC_LIB") or os.path.join(_HERE, "libslc.so")  # SLC_LIB: tuning variants

OK, INVALID_ARGUMENT, INVALID_DATA, STALE, CUDA_ERROR, UNSUPPORTED, FORMAT_ERROR = range(7)
F32, BF16 = 0, 1
MAX_PEERS = 256


class SlcError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} (status {status})")


class Geometry(ctypes.Structure):
    _fields_ = [("block", ctypes.c_int32), ("chunk", ctypes.c_int32), ("k", ctypes.c_int32),
                ("index_bits", ctypes.c_int32)]


class Tensor(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("dims", ctypes.c_int64 * 4)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("total_elems", ctypes.c_int64), ("total_chunks", ctypes.c_int64),
                ("first_chunk", ctypes.c_int64), ("n_chunks", ctypes.c_int64),
                ("shard_elems", ctypes.c_int64), ("record_bytes", ctypes.c_int64),
                ("payload_bytes", ctypes.c_int64), ("n_segments", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32)]


class Segment(ctypes.Structure):
    _fields_ = [("tensor", ctypes.c_int32), ("blocked", ctypes.c_int32), ("tensor_begin", ctypes.c_int64),
                ("n_elems", ctypes.c_int64), ("shard_offset", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("cols", ctypes.c_int64), ("first_chunk", ctypes.c_int64), ("n_chunks", ctypes.c_int64)]


class PayloadHdr(ctypes.Structure):
    _fields_ = [("magic", ctypes.c_char * 4), ("version", ctypes.c_uint32), ("geom", Geometry),
                ("base_round", ctypes.c_uint64), ("peer_id", ctypes.c_uint8 * 16),
                ("layout_digest", ctypes.c_uint8 * 32), ("first_chunk", ctypes.c_int64),
                ("n_chunks", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: the CUDA extension must be built "
                           "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    pp = ctypes.POINTER
    sig = {
        "slc_plan_create": (ctypes.c_int, [pp(Geometry), pp(Tensor), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int, ctypes.c_int32, pp(P)]),
        "slc_plan_info_get": (ctypes.c_int, [P, pp(PlanInfo)]),
        "slc_plan_segment": (ctypes.c_int, [P, ctypes.c_int32, pp(Segment)]),
        "slc_record_bytes": (ctypes.c_int64, [pp(Geometry)]),
        "slc_layout_digest": (ctypes.c_int, [pp(Geometry), pp(Tensor), ctypes.c_int32, P]),
        "slc_compress": (ctypes.c_int, [P, P, P, P, ctypes.c_float, P, P]),
        "slc_compress_multi": (ctypes.c_int, [P, P, P, P, ctypes.c_float, P, ctypes.c_int32, P]),
        "slc_peer_copy": (ctypes.c_int, [P, P, P, P, ctypes.c_int32, P]),
        "slc_compress_range": (ctypes.c_int, [P, ctypes.c_int64, ctypes.c_int64, P, P, P, ctypes.c_float, P, P]),
        "slc_decode_aggregate": (ctypes.c_int, [P, P, P, ctypes.c_int32, P, P, P]),
        "slc_outer_update": (ctypes.c_int, [P, P, P, P, P, ctypes.c_int32, P, ctypes.c_float, P]),
        "slc_payload_sqnorm": (ctypes.c_int, [P, P, P, ctypes.c_int32, P, P]),
        "slc_median_norm_weights": (ctypes.c_int, [P, ctypes.c_int32, P, P, P, P]),
        "slc_decode_aggregate_wdev": (ctypes.c_int, [P, P, P, ctypes.c_int32, P, P, P]),
        "slc_outer_update_wdev": (ctypes.c_int, [P, P, P, P, ctypes.c_int32, P, ctypes.c_float, P]),
        "slc_wire_layout": (ctypes.c_int, [P, pp(ctypes.c_int64), pp(ctypes.c_int64)]),
        "slc_wire_encode": (ctypes.c_int, [P, P, P, P]),
        "slc_wire_decode": (ctypes.c_int, [P, P, ctypes.c_int64, P, P]),
        "slc_wire_header_write": (ctypes.c_int, [pp(PayloadHdr), ctypes.c_int64, P]),
        "slc_wire_header_read": (ctypes.c_int, [P, ctypes.c_int64, pp(PayloadHdr), pp(ctypes.c_int64)]),
        "slc_index_rank": (ctypes.c_int, [P, P, P, P]),
        "slc_plan_set_option": (ctypes.c_int, [P, ctypes.c_int32, ctypes.c_int64]),
        "slc_ec_record_bytes": (ctypes.c_int64, [pp(Geometry)]),
        "slc_index_encode": (ctypes.c_int, [P, P, P, P]),
        "slc_index_decode": (ctypes.c_int, [P, P, P, P]),
        "slc_fast_checks": (ctypes.c_int, [P, P, P, ctypes.c_int32, ctypes.c_uint64, P, P, ctypes.c_int32, P, P]),
        "slc_get_status": (ctypes.c_int, [P, ctypes.c_int32]),
        "slc_plan_destroy": (None, [P]),
        "slc_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


_lib = _load()

EXPORTED = ["slc_plan_create", "slc_plan_info_get", "slc_plan_segment", "slc_record_bytes", "slc_layout_digest",
            "slc_compress", "slc_compress_range", "slc_decode_aggregate", "slc_outer_update", "slc_payload_sqnorm",
            "slc_median_norm_weights", "slc_decode_aggregate_wdev", "slc_outer_update_wdev", "slc_wire_layout",
            "slc_wire_encode", "slc_wire_decode", "slc_wire_header_write", "slc_wire_header_read", "slc_get_status",
            "slc_plan_destroy", "slc_status_string", "slc_index_rank", "slc_plan_set_option",
            "slc_fast_checks", "slc_ec_record_bytes", "slc_index_encode", "slc_index_decode", "slc_compress_multi",
            "slc_peer_copy"]

# slc_fast_checks flag bits (include/slc.h)
CHECK_LIVENESS, CHECK_SYNC, CHECK_FINITE, CHECK_NORM = 1, 2, 4, 8

# slc_option (include/slc.h)
OPT_AGG_KERNEL, OPT_AGG_GRID_CAP, OPT_INDEX_CODE = 1, 2, 3
AGG_KERNELS = {"auto": 0, "batch": 1, "pipe": 2, "simple": 3}


def status_string(s: int) -> str:
    return _lib.slc_status_string(int(s)).decode()


def _check(st: int, what: str):
    if st != OK:
        raise SlcError(st, what)


def geometry(block: int = 64, k: int = 64, index_bits: Optional[int] = None) -> Geometry:
    C = block * block
    ib = index_bits if index_bits is not None else max(1, (C - 1).bit_length())
    return Geometry(block, C, k, ib)


def _layout_array(layout: Sequence[Tuple[str, Tuple[int, ...]]]):
    arr = (Tensor * len(layout))()
    for i, (_, shape) in enumerate(layout):
        if not 1 <= len(shape) <= 4:
            raise ValueError(f"tensor {i}: {len(shape)} dims")
        arr[i].ndim = len(shape)
        for j, s in enumerate(shape):
            arr[i].dims[j] = int(s)
    return arr


def record_bytes(geom: Geometry) -> int:
    return int(_lib.slc_record_bytes(ctypes.byref(geom)))


def layout_digest(geom: Geometry, layout) -> bytes:
    arr = _layout_array(layout)
    out = (ctypes.c_uint8 * 32)()
    _check(_lib.slc_layout_digest(ctypes.byref(geom), arr, len(layout), out), "slc_layout_digest")
    return bytes(out)


def _stream_ptr(stream) -> ctypes.c_void_p:
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(getattr(stream, "cuda_stream", stream))


def _dptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class SegmentInfo:
    tensor: int
    blocked: bool
    tensor_begin: int
    n_elems: int
    shard_offset: int
    rows: int
    cols: int
    first_chunk: int
    n_chunks: int


def wire_header_write(hdr: PayloadHdr, total_chunks: int) -> bytes:
    out = (ctypes.c_uint8 * 65)()
    _check(_lib.slc_wire_header_write(ctypes.byref(hdr), total_chunks, out), "slc_wire_header_write")
    return bytes(out)


def wire_header_read(buf: bytes):
    """(header, total_chunks); SlcError(FORMAT_ERROR) on a bad header."""
    h = PayloadHdr()
    n = ctypes.c_int64()
    b = (ctypes.c_uint8 * max(1, len(buf))).from_buffer_copy(bytes(buf) or b"\0")
    _check(_lib.slc_wire_header_read(b, len(buf), ctypes.byref(h), ctypes.byref(n)), "slc_wire_header_read")
    return h, n.value


def make_header(plan: "Plan", peer_id: bytes, base_round: int = 0) -> PayloadHdr:
    h = PayloadHdr()
    h.magic = b"SLC1"
    h.version = 1
    h.geom = plan.geom
    h.base_round = base_round
    pid = bytes(peer_id)[:16].ljust(16, b"\0")
    for i in range(16):
        h.peer_id[i] = pid[i]
    for i, b in enumerate(plan.digest):
        h.layout_digest[i] = b
    h.first_chunk = plan.info.first_chunk
    h.n_chunks = plan.info.n_chunks
    return h


class Plan:
    """slc_plan of shard `rank` of `nranks` of a global layout.  device < 0 ->
    host-only plan (geometry / partition queries, no compute).

    `default_options` ({slc_option: value}) is applied to every new device
    plan (the tests use it to pin one decode implementation)."""

    default_options: dict = {}

    def __init__(self, layout, geom: Optional[Geometry] = None, rank: int = 0, nranks: int = 1,
                 dtype: str = "f32", device: int = 0):
        self.layout = list(layout)
        self.geom = geom if geom is not None else geometry()
        self.dtype = dtype
        self.device = device
        arr = _layout_array(self.layout)
        h = ctypes.c_void_p()
        _check(_lib.slc_plan_create(ctypes.byref(self.geom), arr, len(self.layout), rank, nranks,
                                    BF16 if dtype == "bf16" else F32, device, ctypes.byref(h)), "slc_plan_create")
        self._h = h
        info = PlanInfo()
        _check(_lib.slc_plan_info_get(h, ctypes.byref(info)), "slc_plan_info_get")
        self.info = info
        self.digest = layout_digest(self.geom, self.layout)
        self.segments: List[SegmentInfo] = []
        for i in range(info.n_segments):
            s = Segment()
            _check(_lib.slc_plan_segment(h, i, ctypes.byref(s)), "slc_plan_segment")
            self.segments.append(SegmentInfo(s.tensor, bool(s.blocked), s.tensor_begin, s.n_elems, s.shard_offset,
                                             s.rows, s.cols, s.first_chunk, s.n_chunks))
        self._index_code = False
        if device >= 0:
            for opt, val in Plan.default_options.items():
                self.set_option(opt, val)

    def set_option(self, option: int, value: int) -> None:
        """slc_plan_set_option (OPT_AGG_KERNEL / OPT_AGG_GRID_CAP / OPT_INDEX_CODE)."""
        _check(_lib.slc_plan_set_option(self._h, int(option), int(value)), "slc_plan_set_option")

    # ---- shape helpers
    @property
    def shard_elems(self) -> int:
        return self.info.shard_elems

    @property
    def n_chunks(self) -> int:
        return self.info.n_chunks

    @property
    def record_bytes(self) -> int:
        return self.info.record_bytes

    @property
    def payload_bytes(self) -> int:
        return self.info.payload_bytes

    # ---- the three calls of the hot path
    def compress(self, theta, theta_local, ef, records, beta: float = 0.95, stream=None) -> None:
        """Eq. 1.  theta/theta_local: [shard_elems] f32|bf16, ef: [shard_elems] f32 (in place),
        records: [payload_bytes] uint8 (or any 4-byte aligned buffer of that size)."""
        self._check_dense(theta, theta_local, ef)
        self._check_bytes(records, self.payload_bytes, "records")
        _check(_lib.slc_compress(self._h, _dptr(theta), _dptr(theta_local), _dptr(ef), ctypes.c_float(beta),
                                 _dptr(records), _stream_ptr(stream)), "slc_compress")

    def compress_multi(self, theta, theta_local, ef, records_out: Sequence, beta: float = 0.95, stream=None) -> None:
        """slc_compress writing the records to every buffer of records_out (tensors, or raw device
        addresses as ints for peer mappings); records_out[0] must be a tensor (size-checked)."""
        self._check_dense(theta, theta_local, ef)
        self._check_bytes(records_out[0], self.payload_bytes, "records")
        ptrs = (ctypes.c_void_p * len(records_out))(*[r if isinstance(r, int) else r.data_ptr() for r in records_out])
        _check(_lib.slc_compress_multi(self._h, _dptr(theta), _dptr(theta_local), _dptr(ef), ctypes.c_float(beta),
                                       ptrs, len(records_out), _stream_ptr(stream)), "slc_compress_multi")

    def peer_copy(self, pairs, stream=None) -> None:
        """Rows a8 / a9: copy [(src, dst, nbytes)] (device addresses as ints, peer mappings allowed) in one kernel."""
        n = len(pairs)
        src = (ctypes.c_void_p * max(1, n))(*[int(a) for a, _, _ in pairs])
        dst = (ctypes.c_void_p * max(1, n))(*[int(b) for _, b, _ in pairs])
        nb = (ctypes.c_int64 * max(1, n))(*[int(c) for _, _, c in pairs])
        _check(_lib.slc_peer_copy(self._h, src, dst, nb, n, _stream_ptr(stream)), "slc_peer_copy")

    def compress_range(self, chunk_begin: int, n_chunks: int, theta, theta_local, ef, records, beta: float = 0.95,
                       stream=None) -> None:
        """slc_compress on the shard-local chunks [chunk_begin, chunk_begin + n_chunks) only (row f3);
        full-shard buffers, only that range's elements / records are touched."""
        self._check_dense(theta, theta_local, ef)
        self._check_bytes(records, self.payload_bytes, "records")
        _check(_lib.slc_compress_range(self._h, ctypes.c_int64(chunk_begin), ctypes.c_int64(n_chunks), _dptr(theta),
                                       _dptr(theta_local), _dptr(ef), ctypes.c_float(beta), _dptr(records),
                                       _stream_ptr(stream)), "slc_compress_range")

    def index_rank(self, records, ranks, stream=None) -> None:
        """Row f4 (R#28): colex rank of every chunk's index set, ranks: [n_chunks * 16] int32/uint32
        little-endian limbs.  The first call prepares the plan's binomial table (OPT_INDEX_CODE)."""
        self._check_bytes(records, self.payload_bytes, "records")
        self._check_bytes(ranks, self.n_chunks * 64, "ranks")
        self._prepare_index_code()
        _check(_lib.slc_index_rank(self._h, _dptr(records), _dptr(ranks), _stream_ptr(stream)), "slc_index_rank")

    @property
    def ec_record_bytes(self) -> int:
        return int(_lib.slc_ec_record_bytes(ctypes.byref(self.geom)))

    def _prepare_index_code(self):
        if not self._index_code:
            self.set_option(OPT_INDEX_CODE, 1)
            self._index_code = True

    def index_encode(self, records, ec, stream=None) -> None:
        """Row f4 (R#28): fixed-width records -> entropy-coded records (n_chunks * ec_record_bytes)."""
        self._check_bytes(records, self.payload_bytes, "records")
        self._check_bytes(ec, self.n_chunks * self.ec_record_bytes, "ec")
        self._prepare_index_code()
        _check(_lib.slc_index_encode(self._h, _dptr(records), _dptr(ec), _stream_ptr(stream)), "slc_index_encode")

    def index_decode(self, ec, records, stream=None) -> None:
        """Row f4 (R#28): entropy-coded records -> fixed-width records (greedy colex unranking on the GPU)."""
        self._check_bytes(ec, self.n_chunks * self.ec_record_bytes, "ec")
        self._check_bytes(records, self.payload_bytes, "records")
        self._prepare_index_code()
        _check(_lib.slc_index_decode(self._h, _dptr(ec), _dptr(records), _stream_ptr(stream)), "slc_index_decode")

    def _peer_args(self, records: Sequence, hdrs, weights):
        R = len(records)
        if not 1 <= R <= MAX_PEERS:
            raise ValueError(f"R={R}")
        for r in records:
            self._check_bytes(r, self.payload_bytes, "records")
        ptrs = (ctypes.c_void_p * R)(*[r.data_ptr() for r in records])
        h = None
        if hdrs is not None:
            h = (PayloadHdr * R)(*hdrs)
        w = None
        if weights is not None:
            w = (ctypes.c_float * R)(*[float(x) for x in weights])
        return R, ptrs, h, w

    def decode_aggregate(self, records: Sequence, agg, hdrs=None, weights=None, stream=None,
                         weights_dev=None) -> None:
        """Eq. 2 line 1: agg[shard_elems] f32 <- (1/R) sum_r w_r decode(records[r]).
        weights: host floats; weights_dev: [R] f32 device tensor (e.g. median_norm_weights)."""
        R, ptrs, h, w = self._peer_args(records, hdrs, weights)
        self._check_f32(agg, "agg")
        if weights_dev is not None:
            self._check_f32(weights_dev, "weights_dev", R)
            _check(_lib.slc_decode_aggregate_wdev(self._h, h, ptrs, R, _dptr(weights_dev), _dptr(agg),
                                                  _stream_ptr(stream)), "slc_decode_aggregate_wdev")
            return
        _check(_lib.slc_decode_aggregate(self._h, h, ptrs, R, w, _dptr(agg), _stream_ptr(stream)),
               "slc_decode_aggregate")

    def fast_checks(self, records: Sequence, flags, current_round: int = 0, hdrs=None, sqnorm=None,
                    norm_history=(), stream=None) -> None:
        """Row f2 fast checks: flags [R] int32 device tensor <- CHECK_* bits per peer.
        records[r] may be None (no submission: CHECK_LIVENESS); sqnorm: rank-summed [R, 4] limbs."""
        R = len(records)
        if not 1 <= R <= MAX_PEERS:
            raise ValueError(f"R={R}")
        for r in records:
            if r is not None:
                self._check_bytes(r, self.payload_bytes, "records")
        ptrs = (ctypes.c_void_p * R)(*[0 if r is None else r.data_ptr() for r in records])
        h = None if hdrs is None else (PayloadHdr * R)(*hdrs)
        hist = [float(x) for x in norm_history]
        harr = (ctypes.c_double * max(1, len(hist)))(*hist) if hist else None
        assert flags.numel() >= R and flags.element_size() == 4
        _check(_lib.slc_fast_checks(self._h, h, ptrs, R, ctypes.c_uint64(current_round), _dptr(sqnorm), harr,
                                    len(hist), _dptr(flags), _stream_ptr(stream)), "slc_fast_checks")

    # ---- SLC1 wire format (NEXT row f2)
    def wire_layout(self):
        """(body_bytes, body_offset) of this shard's chunk encodings in the message body."""
        b, o = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.slc_wire_layout(self._h, ctypes.byref(b), ctypes.byref(o)), "slc_wire_layout")
        return b.value, o.value

    def wire_encode(self, records, wire, stream=None) -> None:
        _check(_lib.slc_wire_encode(self._h, _dptr(records), _dptr(wire), _stream_ptr(stream)), "slc_wire_encode")

    def wire_decode(self, wire, records, stream=None) -> None:
        """wire: the shard's body bytes (a shorter buffer -> SlcError(FORMAT_ERROR), nothing read)."""
        self._check_bytes(records, self.payload_bytes, "records")
        nbytes = wire.numel() * wire.element_size()
        _check(_lib.slc_wire_decode(self._h, _dptr(wire), nbytes, _dptr(records), _stream_ptr(stream)),
               "slc_wire_decode")

    # ---- median-norm normalisation (R#20)
    def payload_sqnorm(self, records: Sequence, out, hdrs=None, stream=None) -> None:
        """out: [R, 4] int64 (uint64 limbs) device tensor <- exact ||hatDelta_r||^2 over this shard."""
        R, ptrs, h, _ = self._peer_args(records, hdrs, None)
        assert out.numel() >= 4 * R and out.element_size() == 8
        _check(_lib.slc_payload_sqnorm(self._h, h, ptrs, R, _dptr(out), _stream_ptr(stream)), "slc_payload_sqnorm")

    def median_norm_weights(self, sqnorm, weights, norms=None, stream=None) -> None:
        """weights: [R] f32 device tensor <- lower-median / ||hatDelta_r|| from the (rank-summed) limbs."""
        R = weights.numel()
        _check(_lib.slc_median_norm_weights(self._h, R, _dptr(sqnorm), _dptr(weights), _dptr(norms),
                                            _stream_ptr(stream)), "slc_median_norm_weights")

    def outer_update(self, theta, alpha: float = 1.0, agg=None, records: Optional[Sequence] = None, hdrs=None,
                     weights=None, stream=None, weights_dev=None) -> None:
        """Eq. 2 line 2: theta <- theta - alpha * Delta; agg=None -> fused decode/aggregate/update."""
        self._check_dense(theta)
        if agg is not None:
            self._check_f32(agg, "agg")
        if weights_dev is not None:
            self._check_f32(weights_dev, "weights_dev", len(records))
            R, ptrs, h, _ = self._peer_args(records, hdrs, None)
            _check(_lib.slc_outer_update_wdev(self._h, _dptr(theta), h, ptrs, R, _dptr(weights_dev),
                                              ctypes.c_float(alpha), _stream_ptr(stream)), "slc_outer_update_wdev")
        elif agg is not None:
            _check(_lib.slc_outer_update(self._h, _dptr(theta), _dptr(agg), None, None, 0, None,
                                         ctypes.c_float(alpha), _stream_ptr(stream)), "slc_outer_update")
        else:
            R, ptrs, h, w = self._peer_args(records, hdrs, weights)
            _check(_lib.slc_outer_update(self._h, _dptr(theta), None, h, ptrs, R, w, ctypes.c_float(alpha),
                                         _stream_ptr(stream)), "slc_outer_update")

    def get_status(self, synchronize: bool = True) -> int:
        return int(_lib.slc_get_status(self._h, 1 if synchronize else 0))

    def check(self) -> None:
        _check(self.get_status(True), "device status")

    def _check_dense(self, theta, theta_local=None, ef=None):
        """theta / theta_local in the plan's param dtype, ef fp32; CUDA tensors on the plan's
        device, contiguous, with at least shard_elems elements."""
        import torch
        pdt = torch.bfloat16 if self.dtype == "bf16" else torch.float32
        for name, t, dt in (("theta", theta, pdt), ("theta_local", theta_local, pdt), ("ef", ef, torch.float32)):
            if t is None:
                continue
            if t.dtype != dt:
                raise TypeError(f"{name}: dtype {t.dtype}, plan expects {dt}")
            if not t.is_cuda or t.device.index != self.device:
                raise ValueError(f"{name}: must be a CUDA tensor on cuda:{self.device}")
            if not t.is_contiguous():
                raise ValueError(f"{name}: must be contiguous")
            if t.numel() < self.shard_elems:
                raise ValueError(f"{name}: {t.numel()} < {self.shard_elems} elements")

    def _check_f32(self, t, name, n=None):
        import torch
        n = self.shard_elems if n is None else n
        if t.dtype != torch.float32 or not t.is_cuda or t.device.index != self.device or not t.is_contiguous():
            raise TypeError(f"{name}: must be a contiguous float32 CUDA tensor on cuda:{self.device}")
        if t.numel() < n:
            raise ValueError(f"{name}: {t.numel()} < {n} elements")

    def _check_bytes(self, t, nbytes, name):
        if t.numel() * t.element_size() < nbytes:
            raise ValueError(f"{name}: {t.numel() * t.element_size()} < {nbytes} bytes")
        if not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{name}: must be a CUDA tensor on cuda:{self.device}")

    def close(self):
        if getattr(self, "_h", None):
            _lib.slc_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""Device residency and the small single-purpose device entry points.

`resolve_operands` turns a plan's operand table (trace records or raw
arrays) into 16-byte-aligned CUDA buffers: payloads already in HBM are used
in place, host payloads (numpy, pinned or pageable torch CPU tensors) are
copied up on the current stream.  Everything numeric goes through the
kernels in libtdb200.so; there is no CPU arithmetic fallback.
"""

from __future__ import annotations

import os
import threading

import numpy as np

from . import _native as N


def is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _payload_of(owner):
    return getattr(owner, "payload", owner)


def to_device(x, stream=None):
    """A contiguous, 16-byte-aligned CUDA tensor holding x's values in x's
    own dtype (numpy arrays keep their dtype; f64 stays f64)."""
    import torch
    if is_torch(x) and x.device.type == "cuda":
        # already resident (the common case, called per operand per check):
        # no availability probe
        if not x.is_contiguous():
            x = x.contiguous()
        return x if x.data_ptr() % 16 == 0 else x.clone()
    if not torch.cuda.is_available():
        raise N.NativeError("no CUDA device: the B200 compare path cannot run here")
    if not is_torch(x):
        arr = np.ascontiguousarray(x)
        if arr.dtype not in (np.float32, np.float64, np.float16):
            arr = arr.astype(np.float64)
        x = torch.from_numpy(arr)
    if x.device.type != "cuda":
        x = x.contiguous().to("cuda", non_blocking=x.is_pinned())
    elif not x.is_contiguous():
        x = x.contiguous()
    if x.data_ptr() % 16 != 0:
        x = x.clone()
    return x


_TORCH_DTYPES = None


class Fingerprints:
    """128-bit digests of many device tensors in ONE td_fingerprint launch
    (replica groups whose copies live on different GPUs).

    The item and chunk tables are staged once; run() can be replayed while
    the tensors stay where they are (the bench times it inside the step).
    `out` is an (n, 2) int64 CUDA tensor, written on the launching stream."""

    def __init__(self, tensors, out=None):
        import torch
        self.tensors = [t if t.is_contiguous() else t.contiguous() for t in tensors]
        for t in self.tensors:
            if t.device.type != "cuda":
                raise N.NativeError("Fingerprints: tensors must be CUDA tensors")
        n = len(self.tensors)
        items = np.zeros(n, N.FP_ITEM)
        items["ptr"] = [t.data_ptr() for t in self.tensors]
        items["nbytes"] = [t.numel() * t.element_size() for t in self.tensors]
        chunks = -(-items["nbytes"] // N.FP_CHUNK)
        begin = np.zeros(n + 1, np.int64)
        np.cumsum(chunks, out=begin[1:])
        self.n, self.n_chunks = n, int(begin[-1])
        self.nbytes = int(items["nbytes"].sum())
        self._items = torch.from_numpy(items.view(np.uint8)).to("cuda")
        self._begin = torch.from_numpy(begin).to("cuda")
        # out: (n, 2) int64 digests, accumulated — run() zeroes its own table,
        # a caller-provided one (a slice of a larger digest table) is zeroed
        # by the caller
        self._own = out is None
        self.out = torch.zeros((max(n, 1), 2), dtype=torch.int64, device="cuda") if out is None else out

    def run(self, stream=None):
        import torch
        if self.n:
            if self._own:
                with torch.cuda.stream(stream or torch.cuda.current_stream()):
                    self.out.zero_()
            N.call("td_fingerprint", self._items.data_ptr(), self._begin.data_ptr(), self.n,
                   self.n_chunks, self.out.data_ptr(), N.stream_handle(stream))
        return self.out[:self.n]


def fingerprints(tensors):
    """(n, 2) int64 CUDA tensor of the tensors' byte digests (one launch)."""
    return Fingerprints(tensors).run()


def stage_host_payloads(traces, stream=None) -> dict:
    """Start the H2D copies of every host-resident payload of `traces` and
    return {id(record): CUDA tensor}.  Copies are asynchronous on the current
    stream, so host-side planning overlaps the DMA.  Payloads that are views
    of one pinned storage (a trace arena, see tracestore.pack_pinned) move
    as ONE copy per storage; the device views keep their offsets."""
    import torch
    staged: dict = {}
    arenas: dict = {}
    pageable: list = []
    tensor = torch.Tensor
    for trace in traces:
        for rec in trace.records:
            p = rec.payload
            if isinstance(p, tensor) and p.is_cuda:
                continue                      # resident: nothing to stage
            if id(rec) in staged:
                continue
            if is_torch(p):
                if p.is_pinned():
                    st = p.untyped_storage()
                    entry = arenas.get(st.data_ptr())
                    if entry is None:
                        # a new arena: its DMA starts now, before the rest of
                        # the records are even looked at
                        host = torch.empty(0, dtype=torch.uint8).set_(st)
                        dev = torch.empty(host.numel(), dtype=torch.uint8, device="cuda")
                        dev.copy_(host, non_blocking=True)
                        entry = arenas[st.data_ptr()] = (dev, [])
                    entry[1].append(rec)
                    continue
            pageable.append(rec)
    if pageable:
        images: dict = {}
        rest = []
        for rec in pageable:
            p = rec.payload
            hit = _image_of(p) if (not is_torch(p) and p.dtype == np.float32
                                   and p.flags.c_contiguous) else None
            if hit is None:
                rest.append(rec)
            else:
                image, off = hit
                images.setdefault(id(image), (image, []))[1].append((rec, off, p.nbytes))
        for key, (image, items) in list(images.items()):
            # an image mostly not referenced by these traces (a subset of a
            # big file) is cheaper through the staging ring than whole
            if 2 * sum(nb for _, _, nb in items) < image.nbytes:
                rest.extend(rec for rec, _, _ in items)
                del images[key]
        if images:
            staged.update(_stage_images(images))
        if rest:
            staged.update(_stage_pageable(rest))
    for dev, recs in arenas.values():
        dst = dev.untyped_storage()
        for rec in recs:
            p = rec.payload
            view = torch.empty(0, dtype=p.dtype, device="cuda").set_(dst, p.storage_offset(),
                                                                     p.shape, p.stride())
            staged[id(rec)] = view if view.data_ptr() % 16 == 0 else view.clone()
    return staged


# page-locked file images that host traces' numpy payloads view
# (read_trace(path, pin=True)): check() moves an image with one DMA and
# unpacks the payloads on the GPU (td_gather_bytes) — no host copy at all.
# Weak: an image lives as long as its trace's payloads do.
_PINNED_IMAGES = None


def register_pinned_image(buf) -> None:
    """buf: the uint8 numpy array over a pinned host allocation that trace
    payloads view (np.frombuffer keeps it alive as their base, so a weak
    reference to it lives exactly as long as the payloads)."""
    global _PINNED_IMAGES
    import weakref
    if _PINNED_IMAGES is None:
        _PINNED_IMAGES = weakref.WeakValueDictionary()
    _PINNED_IMAGES[buf.__array_interface__["data"][0]] = buf


def _image_of(arr):
    """(image array, byte offset) when the numpy array views a registered
    pinned image, else None."""
    if not _PINNED_IMAGES:
        return None
    addr = arr.__array_interface__["data"][0]
    for base, image in list(_PINNED_IMAGES.items()):
        if base <= addr and addr + arr.nbytes <= base + image.nbytes:
            return image, addr - base
    return None


def _stage_images(groups) -> dict:
    """One DMA per pinned image, then one td_gather_bytes unpacking every
    payload into a 256-byte-aligned device arena."""
    import torch
    staged, plans = {}, []
    for image, items in groups.values():
        table, cursor = [], 0
        for rec, off, nbytes in items:
            cursor = -(-cursor // 256) * 256
            table.append((off, cursor, nbytes))
            cursor += nbytes
        # range tables cross before any image: a pageable copy queued behind
        # an image DMA would hold the host until the image had landed
        plans.append((image, items, table, cursor, torch.tensor(table, dtype=torch.int64).to("cuda")))
    for image, items, table, cursor, ranges in plans:
        dev = torch.from_numpy(image).to("cuda", non_blocking=True)
        arena = torch.empty(max(cursor, 16), dtype=torch.uint8, device="cuda")
        N.call("td_gather_bytes", dev.data_ptr(), arena.data_ptr(), ranges.data_ptr(), len(table),
               N.stream_handle())
        for (rec, _, nbytes), (_, dst, _) in zip(items, table):
            p = rec.payload
            staged[id(rec)] = arena[dst:dst + nbytes].view(torch.float32).view(p.shape)
        # the device image is freed once the gather has consumed it (stream order)
        del dev
    return staged


# pageable host payloads (numpy traces, e.g. read_trace() on the host, as a
# reference user has them) cross PCIe through a ring of pinned staging
# buffers: host threads fill buffer k+1 (parallel memcpy, the GIL released
# inside numpy's copy) while buffer k's DMA runs on a copy stream; every
# payload lands 256-byte aligned in one device arena.  Small totals go per
# record (to_device).
_STAGE_CHUNK = 64 << 20
_STAGE_RING = 4
_STAGE_MIN = 64 << 20
_STAGING = None


_STAGING_LOCK = threading.Lock()


def _stage_pageable(records) -> dict:
    # one ring per process: concurrent check() calls take turns on it
    with _STAGING_LOCK:
        return _stage_pageable_locked(records)


def _stage_pageable_locked(records) -> dict:
    import concurrent.futures
    import torch
    global _STAGING
    flat, kinds = [], []                      # raw bytes per payload, (torch dtype, shape)
    for rec in records:
        p = rec.payload
        if is_torch(p):
            t = p.detach().contiguous()
            flat.append(t.reshape(-1).view(torch.uint8).numpy() if t.numel() else np.zeros(0, np.uint8))
            kinds.append((t.dtype, tuple(t.shape)))
        else:
            a = np.ascontiguousarray(p)
            dt = _TORCH_DTYPE_OF_NP.get(a.dtype.str)
            if dt is None:
                a = a.astype(np.float64)
                dt = "float64"
            flat.append(a.reshape(-1).view(np.uint8))
            kinds.append((getattr(torch, dt), a.shape))
    total = 0
    offsets = []
    for a in flat:
        total = -(-total // 256) * 256
        offsets.append(total)
        total += a.nbytes
    if total < _STAGE_MIN:
        return {id(rec): to_device(rec.payload) for rec in records}
    dev = torch.cuda.current_device()
    if _STAGING is None or _STAGING[4] != dev:
        bufs = [torch.empty(_STAGE_CHUNK, dtype=torch.uint8).pin_memory() for _ in range(_STAGE_RING)]
        pool = concurrent.futures.ThreadPoolExecutor(
            max_workers=int(os.environ.get("TD_STAGE_THREADS", min(8, os.cpu_count() or 1))))
        _STAGING = (bufs, [None] * _STAGE_RING, pool, torch.cuda.Stream(), dev)
    bufs, events, pool, copy_stream, _ = _STAGING
    arena = torch.empty(max(total, 16), dtype=torch.uint8, device="cuda")
    copy_stream.wait_stream(torch.cuda.current_stream())
    item, inner, k = 0, 0, 0
    while item < len(flat):
        slot = k % _STAGE_RING
        if events[slot] is not None:
            events[slot].synchronize()           # its previous DMA has drained
        host = bufs[slot].numpy()
        pieces, fill = [], 0                     # (src array slice, staging offset, arena offset)
        dst0 = offsets[item] + inner
        while item < len(flat) and fill < _STAGE_CHUNK:
            src = flat[item]
            start = offsets[item] + inner
            if start != dst0 + fill:             # alignment gap: flush this buffer here
                break
            n = min(src.nbytes - inner, _STAGE_CHUNK - fill)
            pieces.append((src[inner:inner + n], fill))
            fill += n
            inner += n
            if inner == src.nbytes:
                item, inner = item + 1, 0
        if fill == 0:                            # gap before the next payload: restart the buffer there
            dst0 = offsets[item] + inner
            continue
        list(pool.map(lambda pc: np.copyto(host[pc[1]:pc[1] + pc[0].nbytes], pc[0]),
                      _split_pieces(pieces, 8 << 20)))
        with torch.cuda.stream(copy_stream):
            arena[dst0:dst0 + fill].copy_(bufs[slot][:fill], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        events[slot] = ev
        k += 1
    torch.cuda.current_stream().wait_stream(copy_stream)
    staged = {}
    for rec, a, (dt, shape), off in zip(records, flat, kinds, offsets):
        staged[id(rec)] = arena[off:off + a.nbytes].view(dt).view(shape)
    return staged


_TORCH_DTYPE_OF_NP = {"<f4": "float32", "<f8": "float64", "<f2": "float16"}


def _split_pieces(pieces, size):
    """Cut (array, staging offset) copy pieces into <= size parts for the pool."""
    out = []
    for arr, off in pieces:
        for s in range(0, arr.nbytes, size):
            out.append((arr[s:s + size], off + s))
    return out


def resolve_operands(operands, dtypes=None, staged: dict | None = None) -> tuple[np.ndarray, list]:
    """(device addresses as uint64 array, keep-alive list of tensors).

    dtypes[k], when given, is the td_dtype operand k must be presented as;
    a differing payload is widened on the device (exact: bf16/f16 < f32 < f64).
    staged: device copies already in flight (stage_host_payloads)."""
    global _TORCH_DTYPES
    import torch
    if _TORCH_DTYPES is None:
        _TORCH_DTYPES = {N.F32: torch.float32, N.BF16: torch.bfloat16,
                         N.F16: torch.float16, N.F64: torch.float64}
    fast = _resolve_resident(operands, dtypes, staged)
    if fast is not None:
        return fast
    keep = []
    ptrs = np.zeros(len(operands), np.uint64)
    memo: dict = {}
    for k, owner in enumerate(operands):
        t = memo.get(id(owner))
        if t is None and staged is not None:
            t = staged.get(id(owner))
        if t is None:
            dev = getattr(owner, "device_payload", None)
            t = dev() if dev is not None else to_device(_payload_of(owner))
            memo[id(owner)] = t
        if dtypes is not None and N.dtype_code(t) != dtypes[k]:
            t = t.to(_TORCH_DTYPES[dtypes[k]])
        keep.append(t)
        ptrs[k] = t.data_ptr()
    return ptrs, keep


def _resolve_resident(operands, dtypes, staged):
    """resolve_operands when every operand is a record whose payload is
    already a contiguous CUDA tensor of the wanted dtype (device-resident
    traces: torchtap captures, read_trace(device="cuda")): pointers in one
    pass, alignment checked in bulk.  None when any operand needs the general
    path (host payload, staged copy, widening, misalignment)."""
    if staged or dtypes is None:
        return None
    ext = N.host_ext()
    if ext is not None:
        got = ext.resident_ptrs(operands, bytes(dtypes))
        if got is None:
            return None
        return np.frombuffer(got[0], dtype=np.uint64).copy(), got[1]
    return _resolve_resident_py(operands, dtypes)


def _resolve_resident_py(operands, dtypes):
    import torch
    try:
        payloads = [o.payload for o in operands]
    except AttributeError:
        return None
    want = [_TORCH_DTYPES[d] for d in dtypes]
    for t, w in zip(payloads, want):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype is w and t.is_contiguous()):
            return None
    ptrs = np.fromiter((t.data_ptr() for t in payloads), dtype=np.uint64, count=len(payloads))
    if len(ptrs) and (ptrs % 16).any():
        return None
    return ptrs, payloads


class _Raw:
    """A bare array presented as a one-box identity-mapped record."""

    __slots__ = ("tensor", "dtype_code", "shape", "mapping", "replica_group_size")

    def __init__(self, tensor, replicas: int = 1):
        from .canonical import identity_mapping
        self.tensor = tensor
        self.dtype_code = N.dtype_code(tensor)
        self.shape = tuple(tensor.shape)
        self.mapping = identity_mapping(self.shape)
        self.replica_group_size = replicas

    def device_payload(self):
        return self.tensor


def _one_group(ident, records, numeric):
    from .plan import GroupMeta, IdMeta
    meta = IdMeta(ident=ident, exec_index=0, global_shape=records[0].shape)
    meta.groups.append(GroupMeta(records=list(records), declared_detail=None, numeric=numeric))
    return meta


_REL_ERR_WORK: dict = {}
_REL_ERR_LOCK = threading.Lock()


def pair_sums(ta, tb) -> tuple[float, float, float]:
    """(sum (a-b)^2, sum a^2, rel_err) of two contiguous same-dtype CUDA
    tensors: td_rel_err, one launch and one 24-byte D2H."""
    import torch
    dev = ta.device
    # the kernel's partials + ticket are per (device, stream): launches on
    # one stream are ordered, so they never share a workspace concurrently;
    # the 3-double result is per call
    stream = torch.cuda.current_stream(dev)
    key = (dev, stream.cuda_stream)
    with _REL_ERR_LOCK:
        work = _REL_ERR_WORK.get(key)
        if work is None:
            work = _REL_ERR_WORK[key] = torch.zeros(N.REL_ERR_WORK_BYTES, dtype=torch.uint8, device=dev)
    out = torch.empty(3, dtype=torch.float64, device=dev)
    N.call("td_rel_err", ta.data_ptr(), tb.data_ptr(), N.dtype_code(ta), ta.numel(),
           work.data_ptr(), out.data_ptr(), N.stream_handle(stream))
    d2, a2, rel = out.tolist()
    return d2, a2, rel


def rel_err_pair(a, b) -> float:
    """rel_err_arrays(a, b) on the GPU: ||a - b|| / ||a|| with the reference's
    zero conventions (tensor.py:158-167).  Shapes must already agree.

    Same-dtype operands take td_rel_err (one launch, one 24-byte D2H);
    mixed dtypes go through a one-id plan (widening in the compare pass)."""
    from .plan import Plan, PlanEntry
    ta, tb = to_device(a).reshape(-1), to_device(b).reshape(-1)
    if ta.dtype == tb.dtype:
        return pair_sums(ta, tb)[2]
    ra, rb = _Raw(ta), _Raw(tb)
    plan = Plan([PlanEntry("pair", x=_one_group("pair", [ra], False),
                           y=_one_group("pair", [rb], False), x_rep=False, y_rep=False)])
    ptrs, keep = resolve_operands(plan.operands, plan.operand_dtypes)
    idres, _, _ = plan.run(ptrs)
    return float(idres["observed"][0])


def replica_worst(copies) -> tuple[float, int | None]:
    """(worst, index) of max_i rel_err(copy0, copy_i), strict > so NaN never
    wins (canonical.py:236-242); computed by td_segnorm + td_verdict."""
    from .plan import Plan, PlanEntry
    raws = [_Raw(to_device(c).reshape(-1), replicas=len(copies)) for c in copies]
    worst, index = 0.0, None
    # chunks of at most MAX_Z extra copies, each re-reading copy 0 once
    for k in range(1, len(raws), N.MAX_Z):
        chunk = [raws[0]] + raws[k:k + N.MAX_Z]
        plan = Plan([PlanEntry("replicas", x=None, y=_one_group("replicas", chunk, True),
                               x_rep=False, y_rep=True)])
        ptrs, keep = resolve_operands(plan.operands, plan.operand_dtypes)
        _, gres, _ = plan.run(ptrs, replica_eps=float("inf"))
        w, i = float(gres["worst"][0]), int(gres["worst_index"][0])
        if i > 0 and w > worst:
            worst, index = w, k + i - 1
    return worst, index


def merge_boxes(shards, global_shape):
    """td_box_gather: assemble the merged f64 tensor on the device."""
    import torch
    from .plan import _blocks
    out = torch.zeros(tuple(global_shape), dtype=torch.float64, device="cuda")
    gstrides = out.stride() if out.dim() else ()
    for mapping, data in shards:
        src = to_device(data)
        code = N.dtype_code(src)
        rows = []
        for loc, glob in mapping.pairs:
            for so, do, r, c, rs, ds in _blocks(loc.extents, loc.start, mapping.local_shape,
                                                glob.start, tuple(global_shape)):
                rows.append((so, do, r, c, rs, ds))
        if not rows:
            continue
        boxes = torch.tensor(np.array(rows, np.int64).reshape(-1), dtype=torch.int64).to("cuda")
        for k in range(0, len(rows), 65535):
            n = min(65535, len(rows) - k)
            N.call("td_box_gather", src.data_ptr(), code, out.data_ptr(),
                   boxes.data_ptr() + 8 * 6 * k, n, N.stream_handle())
    return out

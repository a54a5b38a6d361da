"""Differential fuzzing of the TTRC path on random traces:
random record counts, shapes (empty, odd sizes that leave payloads
misaligned in the file), shard maps, replica sizes, module names and
headers.  Per case:
  * trace_to_bytes of the device trace (device file image) == of the same
    trace on the host == write_trace's file (device image path) byte for byte;
  * the oracle's independent reader parses that image into the same ids,
    rank metas, maps, replica sizes and f32 payloads;
  * read_trace(device="cuda") and the host reader give back the same
    records, payload bits included;
  * a random truncation or a corrupted magic / length raises the product's
    FormatError where the oracle's reader fails too.

    python tools/fuzz_ttrc.py [--cases 300] [--seed 0]      (GPU)
"""
import argparse
import json
import os
import random
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def random_trace(rnd, device):
    import torch
    from paper_2506_09280_b200.canonical import CanonicalId, ShardMapping, SliceBox, TensorKind, identity_mapping
    from paper_2506_09280_b200.tracestore import RankMeta, Trace, TraceRecord
    header = {"digest": f"d{rnd.randrange(1000)}", "mode": rnd.choice(["cascade", "module"]),
              "note": "x" * rnd.randrange(0, 7)}
    t = Trace(header=header)
    for k in range(rnd.randrange(0, 12)):
        # (no 0-d records: the reference's TraceRecord widens a 0-d host
        # payload to shape (1,) and rejects it, and so does the host reader here)
        ndim = rnd.choice([1, 1, 2, 2, 3])
        shape = tuple(rnd.choice([0, 1, 3, 5, 8, 17]) if rnd.random() < 0.15 else rnd.choice([1, 2, 7, 16, 33, 64])
                      for _ in range(ndim))
        x = torch.randn(shape, device=device)
        if rnd.random() < 0.3 and x.numel():
            x.view(-1)[rnd.randrange(x.numel())] = rnd.choice([float("nan"), float("inf"), -0.0, 1e-40])
        if ndim == 2 and shape[1] and rnd.random() < 0.5:
            g = (shape[0], shape[1] * 2)
            c0 = rnd.choice([0, shape[1]])
            mapping = ShardMapping(shape, g, ((SliceBox(((0, shape[0]), (0, shape[1]))),
                                               SliceBox(((0, shape[0]), (c0, c0 + shape[1])))),))
        else:
            mapping = identity_mapping(shape)
        ident = CanonicalId(rnd.randrange(3), rnd.randrange(4), rnd.choice(list(TensorKind)),
                            f"model.layers.{rnd.randrange(40)}.mod{'_' * rnd.randrange(3)}{k}")
        t.records.append(TraceRecord(ident, RankMeta(*(rnd.randrange(3) for _ in range(6))), mapping,
                                     rnd.choice([1, 1, 2, 4]), x, rnd.choice(["Linear", "Norm", "X" * 9])))
    return t


def same_records(a, b) -> bool:
    import torch
    if a.header != b.header or len(a.records) != len(b.records):
        return False
    for x, y in zip(a.records, b.records):
        if (x.id != y.id or x.rank_meta != y.rank_meta or x.mapping.signature() != y.mapping.signature()
                or x.replica_group_size != y.replica_group_size or x.module_class != y.module_class):
            return False
        px = torch.as_tensor(x.payload).float().cpu().contiguous().view(torch.int32)
        py = torch.as_tensor(y.payload).float().cpu().contiguous().view(torch.int32)
        if px.shape != py.shape or not torch.equal(px, py):
            return False
    return True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    from paper_2506_09280_b200.errors import FormatError
    from paper_2506_09280_b200.tracestore import Trace, TraceRecord, read_trace, trace_from_bytes, trace_to_bytes, \
        write_trace
    from oracle import traindiff_oracle as O
    rnd = random.Random(args.seed)
    t0 = time.time()
    stats = {"cases": 0, "records": 0, "bytes": 0, "corrupt_rejected": 0}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "t.ttrc")
        for k in range(args.cases):
            dev = random_trace(rnd, "cuda")
            host = Trace(header=dict(dev.header),
                         records=[TraceRecord(r.id, r.rank_meta, r.mapping, r.replica_group_size,
                                              r.payload.cpu().numpy(), r.module_class) for r in dev.records])
            img = trace_to_bytes(dev)
            assert img == trace_to_bytes(host), f"case {k}: device image != host image"
            write_trace(dev, path)
            with open(path, "rb") as fh:
                assert fh.read() == img, f"case {k}: write_trace != trace_to_bytes"
            # the file keeps local shapes and box pairs; the global shape read
            # back is the boxes' hull (as the reference reader derives it)
            parsed = trace_from_bytes(img)
            header, orecs = O.read_ttrc(img)
            assert header == dev.header == parsed.header and len(orecs) == len(dev.records), f"case {k}: header"
            for r, o, q in zip(dev.records, orecs, parsed.records):
                assert o.ident == r.id.encode() == q.id.encode(), f"case {k}: ids"
                assert o.rank == r.rank_meta.as_tuple() == q.rank_meta.as_tuple(), f"case {k}: rank"
                assert o.local_shape == r.mapping.local_shape == q.mapping.local_shape, f"case {k}: local shape"
                assert o.global_shape == q.mapping.global_shape, f"case {k}: hull"
                assert o.pairs == q.mapping.pairs_bounds == r.mapping.pairs_bounds, f"case {k}: boxes"
                assert o.replica == r.replica_group_size == q.replica_group_size, f"case {k}: replica"
                assert o.module_class == r.module_class == q.module_class, f"case {k}: class"
                want = r.payload.float().cpu().numpy().reshape(-1).view("<i4")
                assert (o.payload.reshape(-1).view("<i4") == want).all(), f"case {k}: payload"
            for device in ("cuda", None):
                assert same_records(read_trace(path, device=device), parsed), f"case {k}: read_trace({device})"
                assert same_records(trace_from_bytes(img, device=device), parsed), f"case {k}: trace_from_bytes"
            # corruption: truncation, bad magic, an inflated header length
            bad = bytearray(img)
            how = rnd.choice(["truncate", "magic", "length"])
            if how == "truncate" and len(bad) > 1:
                bad = bad[:rnd.randrange(1, len(bad))]
            elif how == "magic":
                bad[0] ^= 0xFF
            else:
                bad[8:12] = (len(bad) + 100).to_bytes(4, "little")
            oracle_ok = True
            try:
                O.read_ttrc(bytes(bad))
            except Exception:             # noqa: BLE001
                oracle_ok = False
            for device in ("cuda", None):
                try:
                    trace_from_bytes(bytes(bad), device=device)
                    ours_ok = True
                except FormatError:
                    ours_ok = False
                assert ours_ok == oracle_ok, f"case {k}: corrupt ({how}) accepted={ours_ok} oracle={oracle_ok}"
            stats["corrupt_rejected"] += not oracle_ok
            stats["cases"] += 1
            stats["records"] += len(dev.records)
            stats["bytes"] += len(img)
    stats["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(stats))


if __name__ == "__main__":
    main()

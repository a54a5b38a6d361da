"""Index-map parity: the ported emission rules produce,
for every layout of the reference's 60-layout grid, exactly the records the
reference emulator traced — same ids in the same order, same RankMeta,
replica sizes, module classes and ShardMapping signatures."""

from paper_2506_09280_b200.layout import (GPT2_MEDIUM, ModelShape, ParallelConfig,
                                          emit_records, piece_positions, seq_pieces, sub_pieces)


def _shape(model):
    return ModelShape(layers=model["layers"], d_model=model["d_model"], n_heads=model["n_heads"],
                      d_ff=model["d_ff"], seq_len=model["seq_len"], vocab=model["vocab"])


def test_emission_matches_reference_over_layout_grid(layouts):
    assert len(layouts) == 60
    for lay in layouts:
        p = lay["parallel"]
        pcfg = ParallelConfig(dp=p["dp"], tp=p["tp"], pp=p["pp"], vp=p["vp"], cp=p["cp"],
                              sp=p["sp"], microbatches=p["microbatches"])
        got = emit_records(_shape(lay["model"]), pcfg)
        want = lay["records"]
        assert len(got) == len(want), p
        for g, w in zip(got, want):
            ident, rank, replica, cls, local, glob, pairs = w
            sig = (tuple(local), tuple(glob),
                   tuple((tuple(map(tuple, l)), tuple(map(tuple, gg))) for l, gg in pairs))
            assert g.ident == ident, p
            assert list(g.rank) == rank, (p, ident)
            assert g.replica == replica, (p, ident)
            assert g.module_class == cls, (p, ident)
            assert g.mapping.signature() == sig, (p, ident)


def test_zigzag_geometry():
    assert seq_pieces(8, 2, 1) == [((0, 2), (2, 4)), ((2, 4), (4, 6))]
    assert piece_positions(seq_pieces(8, 2, 1)) == [2, 3, 4, 5]
    assert sub_pieces(seq_pieces(8, 2, 0), 1, 3) == [((0, 1), (1, 2)), ((1, 2), (6, 7))]


def test_named_shapes_emit():
    recs = emit_records(GPT2_MEDIUM, ParallelConfig(tp=4))
    ids = {r.ident for r in recs}
    assert len(ids) == 1179
    llama = ModelShape(layers=2, d_model=64, n_heads=8, d_ff=128, seq_len=32, vocab=256,
                       n_kv_heads=2, gated_mlp=True, norm_bias=False, position_table=False)
    recs = emit_records(llama, ParallelConfig(tp=2))
    wk = [r for r in recs if r.ident.endswith("attn.wk") and "Param" in r.ident]
    assert wk[0].mapping.global_shape == (64, 16) and wk[0].mapping.local_shape == (64, 8)
    assert any(r.ident.endswith("mlp.w3") for r in recs)

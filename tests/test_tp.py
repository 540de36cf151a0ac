"""Tensor-parallel host logic on CPU: sharding shapes, quantize-then-shard
== shard-then-quantize at group boundaries, and the row-split partial sums reduced by a
real world_size-2 gloo allreduce equal the unsharded GEMM (oracle arithmetic, f64)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_15909_b200 import tp

TINY = tp.LlamaShape("tiny", hidden=512, heads=4, kv_heads=2, head_dim=128, ffn=1024, layers=2)


def full_weights(shape, seed=0):
    rng = np.random.default_rng(seed)
    d = shape.head_dim
    sizes = {"qkv_proj": ((shape.heads + 2 * shape.kv_heads) * d, shape.hidden),
             "attn_out_proj": (shape.hidden, shape.heads * d),
             "ffn_up": (2 * shape.ffn, shape.hidden),
             "ffn_down": (shape.hidden, shape.ffn)}
    return {m: (rng.uniform(-1, 1, s) * (3.0 / s[1]) ** 0.5).astype(np.float32)
            for m, s in sizes.items()}


@pytest.mark.parametrize("world", [1, 2])
def test_shard_shapes_partition_the_weights(world):
    w = full_weights(TINY)
    dims = tp.local_dims(TINY, world)
    rows = {m: [] for m in tp.MODULES}
    for r in range(world):
        for m in tp.MODULES:
            s = tp.shard_module(w[m], m, TINY, r, world)
            assert s.shape == dims.module_shape(TINY, m), (m, r)
            rows[m].append(s)
    # column splits: every full row appears exactly once across ranks
    for m in ("qkv_proj", "ffn_up"):
        got = np.sort(np.concatenate(rows[m]).view([("", np.float32)] * w[m].shape[1]), axis=0)
        ref = np.sort(w[m].view([("", np.float32)] * w[m].shape[1]), axis=0)
        assert np.array_equal(got, ref), m
    # row splits: the K slices tile the full matrix
    for m in ("attn_out_proj", "ffn_down"):
        assert np.array_equal(np.concatenate(rows[m], axis=1), w[m]), m


def test_llama_shapes_shard_at_tp_2_4_8():
    for shape in (tp.LLAMA_8B, tp.LLAMA_70B, tp.LLAMA_405B):
        for world in (1, 2, 4, 8):
            d = tp.local_dims(shape, world)
            assert d.hkv >= 1 and d.attn_cols % 128 == 0 and d.ffn % 128 == 0
    # 70B TP=8 per-rank shards (55.15 MB per layer at W4 g128)
    d = tp.local_dims(tp.LLAMA_70B, 8)
    nbytes = sum(n * k // 2 + n * (k // 128) * 2
                 for n, k in (d.module_shape(tp.LLAMA_70B, m) for m in tp.MODULES))
    assert abs(nbytes / 1e6 - 55.15) < 0.05


@pytest.mark.parametrize("bits", [4, 8])
def test_quantize_then_shard_equals_shard_then_quantize(oracle, bits):
    w = full_weights(TINY, seed=bits)
    for m in tp.MODULES:
        codes, scales = oracle.quantize(w[m], bits, 128)
        for r in range(2):
            sc, ss = oracle.quantize(tp.shard_module(w[m], m, TINY, r, 2), bits, 128)
            if m in ("attn_out_proj", "ffn_down"):  # K split at group boundaries
                k = w[m].shape[1] // 2
                assert np.array_equal(sc, codes[:, r * k:(r + 1) * k]), m
                assert np.array_equal(ss, scales[:, r * (k // 128):(r + 1) * (k // 128)]), m
            else:                                   # row split: rows quantize independently
                assert np.array_equal(sc, tp.shard_module(codes, m, TINY, r, 2)), m
                assert np.array_equal(ss, tp.shard_module(scales, m, TINY, r, 2)), m


TINY8 = tp.LlamaShape("tiny8", hidden=512, heads=8, kv_heads=8, head_dim=128, ffn=2048, layers=1)


@pytest.mark.parametrize("bits,per_channel", [(8, True), (4, False), (8, False)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_quantize_before_shard_partials_sum_to_full(oracle, bits, per_channel, world):
    """quantize the full weight, then shard codes and scales (tp.shard_quantized).
    Row-split shards keep the full row's scale (W8 per-channel: one group per full row), so the
    row-parallel partials summed over ranks equal the unsharded oracle GEMM; column-split
    shards are the full output's columns.  Shard-then-quantize is shown to differ for
    per-channel W8 (its per-shard absmax changes the scales)."""
    w = full_weights(TINY8, seed=world + bits)
    rng = np.random.default_rng(world)
    for m in tp.MODULES:
        n, k = w[m].shape
        g = (1 << (k - 1).bit_length()) if per_channel else 128
        codes, scales = oracle.quantize(w[m], bits, g, k % g != 0)
        data = oracle.pack(codes, bits).reshape(n, k * bits // 8)
        x = rng.uniform(-1, 1, (3, k)).astype(np.float32)
        full = oracle.gemm_oracle_f64(x, codes, g, scales)
        acc = np.zeros_like(full, dtype=np.float64)
        differs = False
        for r in range(world):
            c, s, ks, gs, rg = tp.shard_quantized(data, scales, m, TINY8, r, world, bits, g)
            logical = oracle.unpack(c.ravel(), c.shape[0] * ks, bits).reshape(c.shape[0], ks)
            assert s.shape == (c.shape[0], oracle.groups_per_row(gs, rg, ks)), m
            if m in ("attn_out_proj", "ffn_down"):
                assert np.array_equal(logical, codes[:, r * ks:(r + 1) * ks]), m
                xs = tp.shard_cols(x, r, world)
                acc += oracle.gemm_oracle_f64(xs, logical, gs, s)
                sc, ss = oracle.quantize(tp.shard_cols(w[m], r, world), bits, gs, rg)
                differs |= not np.array_equal(ss, s)
            else:
                assert np.array_equal(logical, tp.shard_module(codes, m, TINY8, r, world)), m
                got = oracle.gemm_oracle_f64(x, logical, gs, s)
                assert np.array_equal(got, tp.shard_module(full.T, m, TINY8, r, world).T), m
        if m in ("attn_out_proj", "ffn_down"):
            assert np.abs(acc - full).max() <= 1e-12 * np.abs(full).max(), (m, world)
            if per_channel:
                assert differs, "per-shard absmax should change some per-channel scales"


def test_row_split_width_must_be_whole_groups():
    with pytest.raises(ValueError):
        tp.local_dims(tp.LlamaShape("bad", 256, 2, 2, 64, 256, 1), 2)  # 64 < group 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
    from oracle import Oracle
    import paper_2505_15909_b200 as rq
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    w = full_weights(TINY, seed=3)
    a = np.random.default_rng(11).uniform(-1, 1, (5, TINY.heads * TINY.head_dim)).astype(np.float32)
    h = np.random.default_rng(12).uniform(-1, 1, (5, TINY.ffn)).astype(np.float32)
    out = {}
    for m, x in (("attn_out_proj", a), ("ffn_down", h)):
        ws = tp.shard_module(w[m], m, TINY, rank, world)
        codes, scales = orc.quantize(ws, 4, 128)
        xs = tp.shard_cols(x, rank, world)
        part = torch.from_numpy(orc.gemm_oracle_f64(xs, codes, 128, scales))
        dist.all_reduce(part)  # the row-parallel sum of the decode layer
        out[m] = part.numpy()
    # column-parallel: each rank's output columns are the full output's columns
    for m in ("qkv_proj", "ffn_up"):
        ws = tp.shard_module(w[m], m, TINY, rank, world)
        codes, scales = orc.quantize(ws, 4, 128)
        x = np.random.default_rng(13).uniform(-1, 1, (5, TINY.hidden)).astype(np.float32)
        out[m] = orc.gemm_oracle_f64(x, codes, 128, scales)
    # every rank resolves the same selective-precision table (plan.cpp:189-224)
    table, _ = rq.plan.resolve("explicit:0 modules:4", 80)
    t = torch.from_numpy(table.astype(np.int64).ravel())
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    out["tables_equal"] = all(torch.equal(g, t) for g in gathered)
    out["q8_slots"] = int((table == 8).sum())
    results[rank] = out
    dist.destroy_process_group()


def test_row_and_column_parallel_over_gloo(oracle):
    world = 2
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    w = full_weights(TINY, seed=3)
    a = np.random.default_rng(11).uniform(-1, 1, (5, TINY.heads * TINY.head_dim)).astype(np.float32)
    h = np.random.default_rng(12).uniform(-1, 1, (5, TINY.ffn)).astype(np.float32)
    x = np.random.default_rng(13).uniform(-1, 1, (5, TINY.hidden)).astype(np.float32)
    for m, inp in (("attn_out_proj", a), ("ffn_down", h)):
        codes, scales = oracle.quantize(w[m], 4, 128)
        ref = oracle.gemm_oracle_f64(inp, codes, 128, scales)
        for r in range(world):
            got = results[r][m]
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (m, r)
    for m in ("qkv_proj", "ffn_up"):
        codes, scales = oracle.quantize(w[m], 4, 128)
        ref = oracle.gemm_oracle_f64(x, codes, 128, scales)
        for r in range(world):
            cols = tp.shard_module(ref.T, m, TINY, r, world).T
            assert np.array_equal(results[r][m], cols), (m, r)
    assert all(results[r]["tables_equal"] for r in range(world))
    assert results[0]["q8_slots"] == 1  # 70B explicit:0 modules:4 -> 1 x q8 + 319 x q4

"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mlstm.h declares,
its pure host functions agree with the paper's numbers, config validation rejects bad input, and
without a GPU it fails loudly (no CPU fallback)."""
import math

import numpy as np
import pytest

import paper_1808_01371_b200 as M
from oracle import mlstm_oracle as O


def test_library_exports_every_header_symbol():
    L = M.lib()
    names = M.header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(M.mlstm._SIGS), "binding and header disagree"


def test_default_config_is_the_papers_4096d_model():
    cfg = M.mlstm_default_config()
    assert (cfg.hidden, cfg.seq_len, cfg.batch, cfg.vocab) == (4096, 256, 256, 256)
    assert cfg.lr0 == 3e-3 and cfg.decay_iters == 100_000
    assert cfg.precision == M.MLSTM_MIXED
    assert M.mlstm_param_count(cfg) == O.param_count(4096, 64) == 86_278_400


def test_pure_functions_match_oracle():
    for it in [0, 1, 777, 50_000, 99_999, 100_000, 123_456]:
        assert M.mlstm_lr_at(3e-3, it, 100_000) == pytest.approx(O.lr_at(3e-3, it, 100_000), abs=1e-18)
    for b in [128, 2048, 4096, 8192, 16384, 32768]:
        assert M.mlstm_scale_lr(5e-4, M.MLSTM_LR_LINEAR, b, 128) == pytest.approx(O.scale_lr(5e-4, "linear", b))
        assert M.mlstm_scale_lr(5e-4, M.MLSTM_LR_SQRT, b, 128) == pytest.approx(O.scale_lr(5e-4, "sqrt", b))
        assert M.mlstm_scale_lr(5e-4, M.MLSTM_LR_NONE, b, 128) == 5e-4
    assert M.mlstm_bpc_from_nats(math.log(256)) == pytest.approx(8.0, abs=1e-14)
    assert M.mlstm_bpc_from_nats(math.log(2)) == pytest.approx(1.0, abs=1e-15)


def test_workspace_size_and_validation():
    small = M.mlstm_default_config(hidden=64, seq_len=16, batch=4)
    assert 0 < M.mlstm_workspace_bytes(small) < 64 << 20
    big = M.mlstm_default_config()
    assert 4e9 < M.mlstm_workspace_bytes(big) < 40e9          # fits a 180 GB B200 many times
    for bad in [dict(hidden=100), dict(embed=48), dict(vocab=255), dict(weight_norm=2), dict(seq_len=0),
                dict(micro_batch=3), dict(precision=7), dict(scale_init=0.5)]:
        cfg = M.mlstm_default_config(**{**dict(hidden=64, seq_len=16, batch=4), **bad})
        with pytest.raises(M.MlstmError) as ei:
            M.mlstm_workspace_bytes(cfg)
        assert ei.value.status == M.MLSTM_EINVAL


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = M.mlstm_default_config(hidden=64, seq_len=16, batch=4)
    with pytest.raises(M.MlstmError) as ei:
        M.mlstm_init(cfg, 256, M.mlstm_workspace_bytes(cfg), 0, None, 0, 1)
    assert ei.value.status == M.MLSTM_ECUDA
    with pytest.raises(RuntimeError):
        M.MLSTM(cfg)


def test_init_argument_errors_have_no_side_effects():
    cfg = M.mlstm_default_config(hidden=64, seq_len=16, batch=4)
    for args in [(0, 1 << 20, 0, None, 0, 1), (256, 1 << 20, 0, None, 2, 2), (256, 1 << 20, 0, None, 0, 2)]:
        with pytest.raises(M.MlstmError) as ei:
            M.mlstm_init(cfg, *args)
        assert ei.value.status == M.MLSTM_EINVAL


@pytest.mark.parametrize("h,B,world,micro", [(4096, 256, 2, 0), (4096, 256, 8, 0), (1024, 128, 4, 0),
                                             (4096, 4096, 2, 1024), (256, 64, 1, 0), (8192, 128, 4, 0)])
def test_allreduce_bucket_plan(h, B, world, micro):
    """The gradient allreduce reduces every element of the canonical fp16 arena
    exactly once, in completion order (buckets never wait on later work than the ones after them): first
    W_dec + b_dec (SURVEY 8(e) "bucket 0", computed before BPTT); on CTA-pair plans the first W_h bucket
    group is units [0, h/2) of each of the four gates (contiguous canonical ranges of h/2 rows), the next
    the other halves; W_mh follows; without overlap (one rank or micro-batches) the plan is the whole
    arena after the backward."""
    cfg = M.mlstm_default_config(hidden=h, embed=64, batch=B, micro_batch=micro)
    P = M.mlstm_param_count(cfg)
    plan = M.mlstm_allreduce_plan(cfg, world)
    cover = np.zeros(P, dtype=np.int32)
    for off, cnt, _ in plan:
        assert cnt > 0 and 0 <= off and off + cnt <= P
        cover[off:off + cnt] += 1
    assert (cover == 1).all()
    afters = [a for _, _, a in plan]
    assert afters == sorted(afters)
    if world == 1 or micro:
        assert plan == [(0, P, 4)]
        return
    e = 64
    off_Wh = 256 * e + h * e + h * h + 4 * h * e      # canonical offset of W_h (include/mlstm.h)
    off_Wmh = 256 * e + h * e
    off_Wdec = off_Wh + 4 * h * h + 4 * h
    assert plan[0] == (off_Wdec, 256 * h + 256, 0)    # W_dec | b_dec, before the backward finishes
    wh = [(o, c) for o, c, a in plan if a in (1, 2)]
    if any(a == 1 for _, _, a in plan):
        first = sorted(o for o, c, a in plan if a == 1)
        assert first == [off_Wh + g * h * h for g in range(4)]                 # gate g, units [0, h/2)
        assert all(c == (h // 2) * h for o, c in wh)
    else:
        assert wh == [(off_Wh, 4 * h * h)]
    assert (off_Wmh, h * h, 3) in plan

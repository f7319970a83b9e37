"""The backend decision table on a machine without a GPU: which keys a stage looks up,
that loaded tables drive the lookups without any timing, and that the digest only depends
on the backend choices (runtime/gemm_tune.py).  Covers the attention backward (K7b) keys
added in round 2."""
import json

import pytest

from paper_2503_01328_b200.runtime import gemm_tune
from paper_2503_01328_b200.runtime.model import ModelConfig


@pytest.fixture(autouse=True)
def clean_table():
    gemm_tune.reset()
    yield
    gemm_tune.reset()


def keys(cfg, **kw):
    return [k for k, _ in gemm_tune.needed_keys(cfg, **kw)]


def test_attention_keys_follow_the_supported_shapes():
    c2 = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=50304)
    k = keys(c2)
    assert gemm_tune.attn_key(4096, 16, 128) in k
    assert gemm_tune.attn_bwd_key(4096, 16, 128) in k
    # forward needs seq % 256, backward seq % 128; head_dim 64 / 128 only
    odd = ModelConfig(n_layers=1, hidden=256, heads=2, seq=384, vocab=512)
    k = keys(odd)
    assert gemm_tune.attn_key(384, 2, 128) not in k and gemm_tune.attn_bwd_key(384, 2, 128) in k
    wide = ModelConfig(n_layers=1, hidden=384, heads=4, seq=512, vocab=512)  # head_dim 96
    assert not any(x.startswith("attn") for x in keys(wide))
    # pinned backends look nothing up
    assert not any(x.startswith("attn") for x in keys(c2, attn="cudnn"))
    assert keys(c2, gemm="cublas", attn="tcgen05") == []


def test_loaded_table_drives_the_choices(tmp_path):
    table = {gemm_tune.attn_key(4096, 16, 128): {"backend": "cudnn", "ours_us": 65.0, "lib_us": 61.0},
             gemm_tune.attn_bwd_key(4096, 16, 128): {"backend": "tcgen05", "ours_us": 184.5, "lib_us": 202.1}}
    path = tmp_path / "table.json"
    path.write_text(json.dumps(table))
    gemm_tune.TABLE.update(table)  # install() also pushes GEMM swizzles into the library
    assert gemm_tune.attn_choice(4096, 16, 128) is False
    assert gemm_tune.attn_bwd_choice(4096, 16, 128) is True
    # a shape missing from the table falls back to the library and is recorded
    assert gemm_tune.attn_bwd_choice(8192, 32, 128) is False
    assert gemm_tune.attn_bwd_key(8192, 32, 128) in gemm_tune.MISSES


def test_digest_depends_on_backends_only():
    gemm_tune.TABLE[gemm_tune.attn_bwd_key(4096, 16, 128)] = {"backend": "tcgen05", "ours_us": 180.0, "lib_us": 200.0}
    d0 = gemm_tune.digest()
    gemm_tune.TABLE[gemm_tune.attn_bwd_key(4096, 16, 128)]["ours_us"] = 999.0
    assert gemm_tune.digest() == d0
    gemm_tune.TABLE[gemm_tune.attn_bwd_key(4096, 16, 128)]["backend"] = "cudnn"
    assert gemm_tune.digest() != d0

"""Non-finite contract: the reference throws std::runtime_error("non-finite
value produced on tape") from every tape op (tape.cpp:29). The engine raises
the same error (ORX_ERUNTIME -> RuntimeError) when a NaN / Inf reaches the
logits of a beam search (device flag set by the pruning kernels) or the host
outputs of encode / teacher-forced scoring / sequence scoring / sampling."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2506_13695_b200 as P  # noqa: E402

LENS = (20, 64, 300)


def _model(precision, name, value):
    cfg = P.PolicyConfig.preset("0.015B")
    w = P.Weights.random(cfg)
    if name is not None:
        x = w.get(name)
        x.flat[7] = value
        w.set(name, x)
    return P.PolicyModel(weights=w, precision=precision, max_users=2, max_width=16)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name,value", [("dec.head1.w", np.inf), ("enc0.attn.wq.w", np.nan),
                                        ("pathway.lifelong.fc1.w", np.inf)])
def test_nonfinite_weight_raises(precision, name, value):
    m = _model(precision, name, value)
    b = P.SynthBatch(1, 0, 2, *LENS)
    with pytest.raises(RuntimeError, match="non-finite value produced on tape"):
        m.beam_search_arrays(b, 16)
    if not name.startswith("dec.head"):  # the encoder output itself is non-finite
        with pytest.raises(RuntimeError, match="non-finite"):
            m.encode_batch(b)
    with pytest.raises(RuntimeError, match="non-finite"):
        m.score_prefixes(b, [0, 1], [[1], [2, 3]])
    with pytest.raises(RuntimeError, match="non-finite"):
        m.sequence_log_prob_batch(b, [0], [[1, 2, 3]])
    # the pipelined path reports it at collect
    m.beam_search_submit(b, 16)
    with pytest.raises(RuntimeError, match="non-finite"):
        m.beam_search_collect()


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_finite_weights_clean(precision):
    """The flag is reset per search: a clean engine after a failing one works."""
    m = _model(precision, None, 0.0)
    b = P.SynthBatch(1, 0, 2, *LENS)
    codes, logp, _ = m.beam_search_arrays(b, 16)
    assert np.isfinite(logp).all()


def test_nonfinite_z_rejected():
    m = _model("fp32", None, 0.0)
    z = np.zeros((1, m.cfg.enc_seq_len(), m.cfg.d_model), dtype=np.float32)
    z[0, 3, 5] = np.inf
    with pytest.raises(RuntimeError, match="non-finite"):
        m.next_logits_batch(z, [0], [[]])

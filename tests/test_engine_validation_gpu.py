"""Request validation inside the engine's staging path (validate_context,
policy.cpp:23-38): the per-record checks run in the parallel packers, and a
failure re-runs the sequential validator so the error raised is the first one
in the reference's order (short -> positive -> lifelong, then user, then record)."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2506_13695_b200 as P  # noqa: E402

N_USERS = 48


@pytest.fixture(scope="module")
def model():
    cfg = P.PolicyConfig.preset("0.015B")
    return P.PolicyModel(cfg, precision="bf16", max_users=N_USERS, max_width=4)


def _users():
    # long enough sequences that the packer uses several worker threads
    cfg = P.PolicyConfig.preset("0.015B")
    return P.SynthBatch(3, 0, N_USERS, cfg.short_len, cfg.positive_len, cfg.lifelong_len).to_contexts()


def test_valid_batch_runs(model):
    codes, logp, n = model.beam_search_arrays(_users(), 4)
    assert codes.shape[0] == N_USERS and (n > 0).all()


@pytest.mark.parametrize("where", [1, N_USERS // 2, N_USERS - 1])
def test_record_errors_from_any_packer(model, where):
    users = _users()
    users[where].lifelong_seq[0].playtime = users[where].lifelong_seq[0].duration + 0.5
    with pytest.raises(ValueError, match="playtime exceeds duration"):
        model.beam_search_arrays(users, 4)
    users = _users()
    users[where].positive_seq[0].labels = 1 << 20
    with pytest.raises(ValueError, match="label bits"):
        model.beam_search_arrays(users, 4)


def test_first_error_in_reference_order(model):
    """A lifelong error in user 0 and a short-sequence error in the last user:
    the sequential order checks every short sequence first."""
    users = _users()
    users[0].lifelong_seq[0].playtime = users[0].lifelong_seq[0].duration + 0.5
    users[-1].short_seq[1].ts = users[-1].short_seq[0].ts - 1
    with pytest.raises(ValueError, match="short sequence not time-ordered"):
        model.beam_search_arrays(users, 4)
    # the engine still serves a valid request afterwards
    codes, _, _ = model.beam_search_arrays(_users(), 4)
    assert codes.shape[0] == N_USERS

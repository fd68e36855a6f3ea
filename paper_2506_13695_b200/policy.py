"""Python mirror of the reference's hot-path API (proj/core policy.hpp,
generation.hpp), backed by the B200 engine in liborx.so.

Reference surface -> here:
  PolicyConfig (policy.hpp:36-85)            -> PolicyConfig (+ presets)
  InteractionFeature/UserContext (15-32)     -> InteractionFeature / UserContext
  PolicyModel(cfg), load, save (59-137,411-443) -> PolicyModel(cfg), PolicyModel.load, .save
  encode_eval (policy.cpp:317-321)           -> PolicyModel.encode_eval / encode_batch
  next_logits_eval (policy.cpp:323-329)      -> PolicyModel.next_logits_eval
  policy_scorer (generation.cpp:163-167)     -> policy_scorer
  GenerationRequest / GeneratedItem          -> same names
  generate / beam_search (generation.cpp:41-88,150-154) -> PolicyModel.generate_batch / generate
  SemanticTrie (trie.hpp)                    -> SemanticTrie (host-side legality lookup)
Errors follow the reference: std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError (OrxError).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from ._lib import (PRECISION, check, lib, orx_beam_out, orx_config, orx_records, orx_trie, orx_user_batch)

_CFG_FIELDS = [f for f, _ in orx_config._fields_]


@dataclass
class PolicyConfig:
    n_layers: int = 4
    d_model: int = 128
    ffn_hidden: int = 256
    n_heads: int = 4
    moe_enabled: bool = False
    n_experts: int = 0
    experts_active: int = 0
    moe_location: str = "decoder"  # or "enc_and_dec"
    expert_round_multiple: int = 128
    n_code_layers: int = 3
    codebook_size: int = 64
    short_len: int = 20
    positive_len: int = 256
    lifelong_len: int = 2000
    n_queries: int = 128
    lifelong_blocks: int = 2
    vid_vocab: int = 4096
    aid_vocab: int = 256
    uid_vocab: int = 1024
    gender_vocab: int = 3
    age_vocab: int = 8
    n_label_flags: int = 5
    use_sid_history: bool = False
    vid_only_features: bool = False
    compress_threshold: int = 8
    moe_bias_update: float = 1e-3
    seed: int = 123

    @staticmethod
    def preset(name: str, **overrides) -> "PolicyConfig":
        c = orx_config()
        check(lib().orx_config_preset(name.encode(), C.byref(c)))
        cfg = PolicyConfig.from_c(c)
        return dataclasses.replace(cfg, **overrides)

    @staticmethod
    def from_c(c: orx_config) -> "PolicyConfig":
        kw = {}
        for f in _CFG_FIELDS:
            v = getattr(c, f)
            if f == "moe_location":
                v = "decoder" if v == 0 else "enc_and_dec"
            elif f in ("moe_enabled", "use_sid_history", "vid_only_features"):
                v = bool(v)
            kw[f] = v
        return PolicyConfig(**kw)

    def to_c(self) -> orx_config:
        c = orx_config()
        for f in _CFG_FIELDS:
            v = getattr(self, f)
            if f == "moe_location":
                v = 0 if v == "decoder" else 1
            setattr(c, f, type(getattr(c, f))(v))
        return c

    def enc_layers(self) -> int:
        return self.n_layers // 2

    def dec_layers(self) -> int:
        return self.n_layers - self.n_layers // 2

    def enc_seq_len(self) -> int:
        return 1 + self.short_len + self.positive_len + self.n_queries

    def expert_hidden(self) -> int:
        return int(lib().orx_config_expert_hidden(C.byref(self.to_c())))


@dataclass
class InteractionFeature:
    vid: int = 0
    sid: List[int] = field(default_factory=list)
    aid: int = 0
    tag: float = 0.0
    ts: float = 0.0
    playtime: float = 0.0
    duration: float = 0.0
    labels: int = 0


@dataclass
class UserContext:
    uid: int = 0
    gender: int = 0
    age_bucket: int = 0
    short_seq: List[InteractionFeature] = field(default_factory=list)
    positive_seq: List[InteractionFeature] = field(default_factory=list)
    lifelong_seq: List[InteractionFeature] = field(default_factory=list)


@dataclass
class GenerationRequest:
    strategy: str = "beam"
    width: int = 8
    constrain_to_trie: bool = False
    temperature: float = 1.0
    top_k: int = 0
    top_p: float = 1.0


def validate_request(req: GenerationRequest) -> None:  # generation.cpp:34-39
    if req.width < 1:
        raise ValueError("generation width must be >= 1")
    if not (0 < req.top_p <= 1.0):
        raise ValueError("top_p must lie in (0,1]")
    if req.top_k < 0:
        raise ValueError("top_k must be >= 1 (or 0 for the full vocabulary)")
    if not req.temperature > 0:
        raise ValueError("temperature must be positive")


@dataclass
class GeneratedItem:
    codes: List[int]
    log_prob: float
    legal: bool = False
    item_ids: List[int] = field(default_factory=list)


class SemanticTrie:
    """Host prefix tree over legal code sequences (trie.hpp:27-62)."""

    def __init__(self, depth: int):
        if depth < 1:
            raise ValueError("trie depth must be >= 1")
        self.depth = depth
        self._leaves: Dict[tuple, List[int]] = {}
        self.version = 0  # bumped by insert(): a PolicyModel re-uploads a changed trie

    def insert(self, codes: Sequence[int], item: int) -> None:
        if len(codes) != self.depth:
            raise ValueError("semantic id length must equal trie depth")
        if any(c < 0 for c in codes):
            raise ValueError("semantic id codes must be non-negative")
        self._leaves.setdefault(tuple(codes), []).append(int(item))
        self.version += 1

    def lookup(self, codes: Sequence[int]) -> Optional[List[int]]:
        return self._leaves.get(tuple(codes)) if len(codes) == self.depth else None

    def item_count(self) -> int:
        return sum(len(v) for v in self._leaves.values())

    def children_of(self, prefix: Sequence[int]) -> List[int]:  # trie.cpp:53-59
        n = len(prefix)
        if n >= self.depth:
            return []
        p = tuple(prefix)
        return sorted({k[n] for k in self._leaves if k[:n] == p})

    def to_csr(self):
        """(child_off, child_code, child_node) int32 arrays over prefix nodes,
        node 0 = root, children in ascending code order (std::map order)."""
        nodes = {(): 0}
        level = [()]
        edges = {0: []}
        for depth in range(self.depth):
            nxt = sorted({k[:depth + 1] for k in self._leaves})
            for pre in nxt:
                nodes[pre] = len(nodes)
                edges[nodes[pre]] = []
                edges[nodes[pre[:-1]]].append((pre[-1], nodes[pre]))
            level = nxt
        off, code, node = [0], [], []
        for n in range(len(nodes)):
            for c, ch in sorted(edges[n]):
                code.append(c)
                node.append(ch)
            off.append(len(code))
        del level
        return (np.asarray(off, dtype=np.int32), np.asarray(code, dtype=np.int32), np.asarray(node, dtype=np.int32))


# ---- user batches ------------------------------------------------------------------

class UserBatch:
    """Owns packed SoA host arrays and exposes them as an orx_user_batch."""

    def __init__(self, users: Sequence[UserContext], n_code_layers: int = 3):
        self.n_users = len(users)
        self._keep = []
        self.c = orx_user_batch()
        self.c.n_users = self.n_users
        self.c.uid = self._arr([u.uid for u in users], np.int32, C.c_int32)
        self.c.gender = self._arr([u.gender for u in users], np.int32, C.c_int32)
        self.c.age_bucket = self._arr([u.age_bucket for u in users], np.int32, C.c_int32)
        for name in ("short_seq", "positive_seq", "lifelong_seq"):
            recs = [getattr(u, name) for u in users]
            setattr(self.c, name, self._records(recs, n_code_layers))

    def _arr(self, values, dtype, ctype):
        a = np.ascontiguousarray(np.asarray(values, dtype=dtype))
        if a.size == 0:
            a = np.zeros(1, dtype=dtype)
        self._keep.append(a)
        return a.ctypes.data_as(C.POINTER(ctype))

    def _records(self, per_user, L) -> orx_records:
        r = orx_records()
        flat = [f for seq in per_user for f in seq]
        r.offsets = self._arr(np.cumsum([0] + [len(s) for s in per_user]), np.int64, C.c_int64)
        r.vid = self._arr([f.vid for f in flat], np.int64, C.c_int64)
        r.aid = self._arr([f.aid for f in flat], np.int32, C.c_int32)
        r.tag = self._arr([f.tag for f in flat], np.float64, C.c_double)
        r.ts = self._arr([f.ts for f in flat], np.float64, C.c_double)
        r.playtime = self._arr([f.playtime for f in flat], np.float64, C.c_double)
        r.duration = self._arr([f.duration for f in flat], np.float64, C.c_double)
        r.labels = self._arr([f.labels for f in flat], np.uint32, C.c_uint32)
        if flat and all(len(f.sid) == L for f in flat):
            r.sid = self._arr([c for f in flat for c in f.sid], np.int32, C.c_int32)
        return r


class SynthBatch:
    """Seeded synthetic users generated natively (csrc/synth_users.hpp)."""

    def __init__(self, seed: int, user_begin: int, n_users: int, n_short: int = 20, n_positive: int = 256,
                 n_lifelong: int = 2000):
        self._h = C.c_void_p()
        check(lib().orx_synth_batch_create(seed, user_begin, n_users, n_short, n_positive, n_lifelong,
                                           C.byref(self._h)))
        self.c = orx_user_batch()
        check(lib().orx_synth_batch_view(self._h, C.byref(self.c)))
        self.n_users = n_users

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orx_synth_batch_destroy(self._h)
            self._h = None

    def to_contexts(self) -> List[UserContext]:
        out = []
        b = self.c
        for u in range(self.n_users):
            ctx = UserContext(uid=b.uid[u], gender=b.gender[u], age_bucket=b.age_bucket[u])
            for name in ("short_seq", "positive_seq", "lifelong_seq"):
                r = getattr(b, name)
                seq = getattr(ctx, name)
                for i in range(r.offsets[u], r.offsets[u + 1]):
                    seq.append(InteractionFeature(vid=r.vid[i], aid=r.aid[i], tag=r.tag[i], ts=r.ts[i],
                                                  playtime=r.playtime[i], duration=r.duration[i],
                                                  labels=r.labels[i]))
            out.append(ctx)
        return out


def _as_batch(users, L):
    if isinstance(users, (UserBatch, SynthBatch)):
        return users
    if isinstance(users, UserContext):
        users = [users]
    return UserBatch(list(users), L)


# ---- model -----------------------------------------------------------------------------

class Weights:
    """Host weights (fp32 copies of the reference's f64 parameters)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @staticmethod
    def random(cfg: PolicyConfig) -> "Weights":
        h = C.c_void_p()
        check(lib().orx_weights_create_random(C.byref(cfg.to_c()), C.byref(h)))
        return Weights(h)

    @staticmethod
    def random_ep(cfg: PolicyConfig, ep_rank: int, ep_world: int, owner=None) -> "Weights":
        """The same seeded weights, materialising only the experts this
        expert-parallel rank computes (contiguous blocks, or per the placement
        `owner` [moe_layers, n_experts]: rank, or -1 = replicated)."""
        h = C.c_void_p()
        if owner is None:
            check(lib().orx_weights_create_random_ep(C.byref(cfg.to_c()), ep_rank, ep_world, C.byref(h)))
        else:
            own = _placement(cfg, owner)
            check(lib().orx_weights_create_random_ep_placed(C.byref(cfg.to_c()), ep_rank, ep_world,
                                                            own.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(h)))
        return Weights(h)

    @staticmethod
    def load(path: str) -> "Weights":
        h = C.c_void_p()
        check(lib().orx_weights_load_grcp(str(path).encode(), C.byref(h)))
        return Weights(h)

    def save(self, path: str) -> None:
        check(lib().orx_weights_save_grcp(self._h, str(path).encode()))

    def config(self) -> PolicyConfig:
        c = orx_config()
        check(lib().orx_weights_config(self._h, C.byref(c)))
        return PolicyConfig.from_c(c)

    def names(self) -> List[str]:
        out = []
        for i in range(lib().orx_weights_count(self._h)):
            name = C.c_char_p()
            check(lib().orx_weights_entry(self._h, i, C.byref(name), None, None, None))
            out.append(name.value.decode())
        return out

    def get(self, name: str) -> np.ndarray:
        idx = C.c_int64()
        check(lib().orx_weights_find(self._h, name.encode(), C.byref(idx)))
        dims = (C.c_int32 * 2)()
        data = C.POINTER(C.c_float)()
        check(lib().orx_weights_entry(self._h, idx.value, None, None, dims, C.byref(data)))
        if not data:  # an expert another expert-parallel rank computes (not materialised here)
            return np.zeros((0, 0), dtype=np.float32)
        n = dims[0] * dims[1]
        return np.ctypeslib.as_array(data, shape=(n,)).reshape(dims[0], dims[1]).copy()

    def set(self, name: str, value: np.ndarray) -> None:
        """Overwrite a named parameter (reference name, e.g. "dec.head0.w")."""
        v = np.ascontiguousarray(np.asarray(value, dtype=np.float32).ravel())
        check(lib().orx_weights_set(self._h, name.encode(), v.ctypes.data_as(C.POINTER(C.c_float)), v.size))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orx_weights_destroy(self._h)
            self._h = None


def moe_layers(cfg: PolicyConfig) -> int:
    """MoE layers in engine order (encoder layers when they are MoE, then decoder layers)."""
    return int(lib().orx_config_moe_layers(C.byref(cfg.to_c())))


def _placement(cfg: PolicyConfig, owner) -> np.ndarray:
    own = np.ascontiguousarray(np.asarray(owner, dtype=np.int32))
    if own.shape != (moe_layers(cfg), cfg.n_experts):
        raise ValueError(f"expert placement must be [moe_layers={moe_layers(cfg)}, n_experts={cfg.n_experts}]")
    return own


def ep_place(load, world: int, max_replicas: int, min_replicas: int = 0):
    """Load-balanced expert placement (csrc/ep_plan.hpp ep_place_balanced)
    from per-layer expert loads [moe_layers, n_experts] (PolicyModel.expert_load):
    returns (owner [moe_layers, n_experts] int32, predicted busiest/mean rank load per layer)."""
    ld = np.ascontiguousarray(np.asarray(load, dtype=np.int64))
    if ld.ndim != 2:
        raise ValueError("load must be [moe_layers, n_experts]")
    owner = np.empty(ld.shape, dtype=np.int32)
    pred = np.empty(ld.shape[0], dtype=np.float64)
    check(lib().orx_ep_place(ld.ctypes.data_as(C.POINTER(C.c_int64)), ld.shape[0], ld.shape[1], world, min_replicas,
                             max_replicas,
                             owner.ctypes.data_as(C.POINTER(C.c_int32)), pred.ctypes.data_as(C.POINTER(C.c_double))))
    return owner, pred


class PolicyModel:
    """Encoder + MoE decoder on one B200 (the engine owns device weights)."""

    def __init__(self, cfg: Optional[PolicyConfig] = None, *, weights: Optional[Weights] = None,
                 precision: str = "fp32", device: int = 0, max_users: int = 16, max_width: int = 128,
                 ep: Optional[tuple] = None, ep_owner=None):
        """ep = (rank, world, unique_id bytes): expert-parallel engine holding
        n_experts / world experts per MoE layer (see dist.ep_unique_id), or the
        experts the placement ep_owner [moe_layers, n_experts] gives this rank
        (rank, or -1 = replicated; the same table on every rank; see ep_place)."""
        if weights is None:
            if cfg is None:
                raise ValueError("PolicyModel needs a config or weights")
            weights = Weights.random(cfg)
        self.weights = weights
        self.cfg = weights.config()
        self.precision = precision
        self.max_users, self.max_width = max_users, max_width
        self._pending = []  # (n_users, width) of submitted, not yet collected beam searches
        self._e = C.c_void_p()
        if ep is None or ep[1] == 1:
            check(lib().orx_engine_create(weights._h, device, PRECISION[precision], max_users, max_width,
                                          C.byref(self._e)))
        else:
            rank, world, uid = ep
            buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
            own = None if ep_owner is None else _placement(self.cfg, ep_owner)
            check(lib().orx_engine_create_ep_placed(
                weights._h, device, PRECISION[precision], max_users, max_width, buf, rank, world,
                None if own is None else own.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(self._e)))

    def expert_load(self, reset: bool = False) -> np.ndarray:
        """Expert-parallel engines: rows routed to each expert of each MoE layer,
        over every rank and call since creation / the last reset
        [moe_layers, n_experts] (identical on every rank; zeros otherwise)."""
        out = np.zeros((moe_layers(self.cfg), self.cfg.n_experts), dtype=np.int64)
        if out.size:
            check(lib().orx_engine_expert_load(self._e, out.ctypes.data_as(C.POINTER(C.c_int64)), int(reset)))
        return out

    @staticmethod
    def load(path: str, **kw) -> "PolicyModel":
        return PolicyModel(weights=Weights.load(path), **kw)

    def save(self, path: str) -> None:
        self.weights.save(path)

    def config(self) -> PolicyConfig:
        return self.cfg

    def __del__(self):
        if getattr(self, "_e", None):
            lib().orx_engine_destroy(self._e)
            self._e = None

    # -- encode ----------------------------------------------------------------------
    def encode_batch(self, users) -> np.ndarray:
        b = _as_batch(users, self.cfg.n_code_layers)
        T, d = self.cfg.enc_seq_len(), self.cfg.d_model
        z = np.empty((b.n_users, T, d), dtype=np.float32)
        check(lib().orx_encode(self._e, C.byref(b.c), z.ctypes.data_as(C.POINTER(C.c_float))))
        return z

    def encode_eval(self, ctx: UserContext) -> np.ndarray:
        return self.encode_batch([ctx])[0]

    # -- teacher-forced logits ---------------------------------------------------------
    def next_logits_batch(self, z_enc: np.ndarray, z_index: Sequence[int], prefixes: Sequence[Sequence[int]]):
        L, V = self.cfg.n_code_layers, self.cfg.codebook_size
        z = np.ascontiguousarray(z_enc, dtype=np.float32)
        if z.ndim == 2:
            z = z[None]
        n = len(prefixes)
        pre = np.full((max(n, 1), L), -1, dtype=np.int32)
        plen = np.zeros(max(n, 1), dtype=np.int32)
        for i, p in enumerate(prefixes):
            if len(p) > L - 1:
                raise ValueError("no prediction head at this position")
            pre[i, :len(p)] = p
            plen[i] = len(p)
        zi = np.ascontiguousarray(np.asarray(z_index, dtype=np.int32).reshape(-1))
        out = np.empty((max(n, 1), V), dtype=np.float32)
        I32 = C.POINTER(C.c_int32)
        check(lib().orx_next_logits(self._e, z.ctypes.data_as(C.POINTER(C.c_float)), z.shape[0], n,
                                    zi.ctypes.data_as(I32), pre.ctypes.data_as(I32), plen.ctypes.data_as(I32),
                                    out.ctypes.data_as(C.POINTER(C.c_float))))
        return out[:n]

    def next_logits_eval(self, z_enc: np.ndarray, prefix: Sequence[int]) -> np.ndarray:
        """Logits (1, V) for the next code after `prefix` (policy.cpp:323-329)."""
        return self.next_logits_batch(z_enc, [0], [list(prefix)])

    def score_prefixes(self, users, user_index: Sequence[int], prefixes: Sequence[Sequence[int]]) -> np.ndarray:
        b = _as_batch(users, self.cfg.n_code_layers)
        L, V = self.cfg.n_code_layers, self.cfg.codebook_size
        n = len(prefixes)
        pre = np.full((max(n, 1), L), -1, dtype=np.int32)
        plen = np.zeros(max(n, 1), dtype=np.int32)
        for i, p in enumerate(prefixes):
            pre[i, :len(p)] = p
            plen[i] = len(p)
        ui = np.ascontiguousarray(np.asarray(user_index, dtype=np.int32))
        out = np.empty((max(n, 1), V), dtype=np.float32)
        I32 = C.POINTER(C.c_int32)
        check(lib().orx_score_prefixes(self._e, C.byref(b.c), n, ui.ctypes.data_as(I32), pre.ctypes.data_as(I32),
                                       plen.ctypes.data_as(I32), out.ctypes.data_as(C.POINTER(C.c_float))))
        return out[:n]

    # -- generation ----------------------------------------------------------------------
    def set_trie(self, trie: "SemanticTrie") -> None:
        """Upload the semantic-ID trie for constrained beam search."""
        off, code, node = trie.to_csr()
        self._trie_keep = (off, code, node)
        I32 = C.POINTER(C.c_int32)
        t = orx_trie(len(off) - 1, off.ctypes.data_as(I32), len(code), code.ctypes.data_as(I32), node.ctypes.data_as(I32))
        check(lib().orx_engine_set_trie(self._e, C.byref(t)))
        self._trie = trie
        self._trie_version = trie.version

    def sequence_log_prob_batch(self, users, user_index: Sequence[int], codes: Sequence[Sequence[int]]) -> np.ndarray:
        """PolicyModel::sequence_log_prob (policy.cpp:297-310) for (user, full code) queries, f64."""
        b = _as_batch(users, self.cfg.n_code_layers)
        L = self.cfg.n_code_layers
        cs = np.ascontiguousarray(np.asarray(codes, dtype=np.int32).reshape(-1, L))
        ui = np.ascontiguousarray(np.asarray(user_index, dtype=np.int32).reshape(-1))
        if cs.shape[0] != ui.shape[0]:
            raise ValueError("one user index per sequence")
        out = np.empty(max(len(ui), 1), dtype=np.float64)
        I32 = C.POINTER(C.c_int32)
        check(lib().orx_sequence_log_prob(self._e, C.byref(b.c), len(ui), ui.ctypes.data_as(I32),
                                          cs.ctypes.data_as(I32), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out[:len(ui)]

    def sample_arrays(self, users, width: int, temperature: float = 1.0, top_k: int = 0, top_p: float = 1.0,
                      seed: int = 0, streams: Optional[Sequence[int]] = None):
        """sample_topk_topp (generation.cpp:90-148) for every user: (codes [U, W, L], log_prob [U, W]);
        user u draws from Rng(seed).split(streams[u]) (default: u)."""
        b = _as_batch(users, self.cfg.n_code_layers)
        L = self.cfg.n_code_layers
        codes = np.empty((b.n_users, width, L), dtype=np.int32)
        logp = np.empty((b.n_users, width), dtype=np.float64)
        n_items = np.empty(b.n_users, dtype=np.int32)
        out = orx_beam_out(codes.ctypes.data_as(C.POINTER(C.c_int32)), logp.ctypes.data_as(C.POINTER(C.c_double)),
                           n_items.ctypes.data_as(C.POINTER(C.c_int32)))
        st = None
        if streams is not None:
            st_arr = np.ascontiguousarray(np.asarray(streams, dtype=np.uint64))
            if st_arr.shape[0] != b.n_users:
                raise ValueError("one stream id per user")
            st = st_arr.ctypes.data_as(C.POINTER(C.c_uint64))
        check(lib().orx_sample(self._e, C.byref(b.c), width, float(temperature), int(top_k), float(top_p),
                               C.c_uint64(seed), st, C.byref(out)))
        return codes, logp

    def beam_search_arrays(self, users, width: int, constrained: bool = False):
        """Batched beam search: (codes [U, W, L] int32, log_prob [U, W] f64, n_items [U]).
        constrained=True expands only children of the trie set by set_trie."""
        b = _as_batch(users, self.cfg.n_code_layers)
        L = self.cfg.n_code_layers
        codes = np.empty((b.n_users, width, L), dtype=np.int32)
        logp = np.empty((b.n_users, width), dtype=np.float64)
        n_items = np.empty(b.n_users, dtype=np.int32)
        out = orx_beam_out(codes.ctypes.data_as(C.POINTER(C.c_int32)), logp.ctypes.data_as(C.POINTER(C.c_double)),
                           n_items.ctypes.data_as(C.POINTER(C.c_int32)))
        fn = lib().orx_beam_search_constrained if constrained else lib().orx_beam_search
        check(fn(self._e, C.byref(b.c), width, C.byref(out)))
        return codes, logp, n_items

    def beam_search_submit(self, users, width: int) -> None:
        """Pipelined form of beam_search_arrays: stage + launch without waiting
        (at most two in flight); beam_search_collect returns the oldest."""
        b = _as_batch(users, self.cfg.n_code_layers)
        check(lib().orx_beam_search_submit(self._e, C.byref(b.c), width))
        self._pending.append((b.n_users, width))

    def beam_search_collect(self):
        if not self._pending:
            raise ValueError("no beam search in flight")
        n_users, width = self._pending[0]
        L = self.cfg.n_code_layers
        codes = np.empty((n_users, width, L), dtype=np.int32)
        logp = np.empty((n_users, width), dtype=np.float64)
        n_items = np.empty(n_users, dtype=np.int32)
        out = orx_beam_out(codes.ctypes.data_as(C.POINTER(C.c_int32)), logp.ctypes.data_as(C.POINTER(C.c_double)),
                           n_items.ctypes.data_as(C.POINTER(C.c_int32)))
        rc = lib().orx_beam_search_collect(self._e, C.byref(out))
        self._pending.pop(0)  # the engine retires the request even when it fails (e.g. non-finite)
        check(rc)
        return codes, logp, n_items

    def generate_batch(self, users, req: GenerationRequest, trie: Optional[SemanticTrie] = None, seed: int = 0,
                       streams: Optional[Sequence[int]] = None) -> List[List[GeneratedItem]]:
        validate_request(req)
        if req.strategy != "beam":  # sample_topk_topp (generation.cpp:90-148)
            codes, logp = self.sample_arrays(users, req.width, req.temperature, req.top_k, req.top_p, seed, streams)
            out = []
            for u in range(codes.shape[0]):
                items = []
                for s_ in range(req.width):
                    c = [int(x) for x in codes[u, s_]]
                    ids = trie.lookup(c) if trie is not None else None
                    items.append(GeneratedItem(codes=c, log_prob=float(logp[u, s_]), legal=ids is not None,
                                               item_ids=list(ids or [])))
                out.append(items)
            return out
        if req.constrain_to_trie:
            if trie is None or trie.item_count() == 0:
                raise ValueError("constrained beam search over an empty trie")  # generation.cpp:44-45
            if getattr(self, "_trie", None) is not trie or self._trie_version != trie.version:
                self.set_trie(trie)
        codes, logp, n_items = self.beam_search_arrays(users, req.width, constrained=req.constrain_to_trie)
        out = []
        for u in range(codes.shape[0]):
            items = []
            for b in range(int(n_items[u])):
                c = [int(x) for x in codes[u, b]]
                ids = trie.lookup(c) if trie is not None else None
                items.append(GeneratedItem(codes=c, log_prob=float(logp[u, b]), legal=ids is not None,
                                           item_ids=list(ids or [])))
            out.append(items)
        return out

    def generate(self, ctx: UserContext, req: GenerationRequest, trie: Optional[SemanticTrie] = None,
                 seed: int = 0, stream: int = 0) -> List[GeneratedItem]:
        return self.generate_batch([ctx], req, trie, seed, [stream])[0]

    def stats(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().orx_engine_stats(self._e, C.byref(a), C.byref(b), C.byref(c)))
        return {"launches": a.value, "h2d_bytes": b.value, "d2h_bytes": c.value}


def policy_scorer(model: PolicyModel, z_enc: np.ndarray):
    """StepScorer closure (generation.cpp:163-167): prefix -> logits (1, V)."""
    z = np.ascontiguousarray(z_enc, dtype=np.float32)
    return lambda prefix: model.next_logits_eval(z, prefix)


def compress_lifelong_batch(offsets, vid, aid, tag, ts, playtime, duration, labels, content, rng_seeds,
                            threshold: int = 8, max_out: int = 2000, sid=None, n_code_layers: int = 3,
                            device: int = 0):
    """compress_lifelong (policy.cpp:447-510) for a batch of raw histories on
    the GPU (hierarchical K-means, bit-identical to the reference's f64 code).
    Inputs are flat per-record arrays with user offsets; content is
    [n_records, D] f64; rng_seeds[u] seeds user u's Rng. Returns a dict of
    the compressed flat arrays (last min(n_u, max_out) records per user)."""
    from ._lib import orx_records, orx_records_out
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    U = len(off) - 1
    cnt = np.diff(off)
    n_out = int(np.minimum(cnt, max_out).sum())
    arr = {"vid": np.ascontiguousarray(vid, dtype=np.int64), "aid": np.ascontiguousarray(aid, dtype=np.int32),
           "tag": np.ascontiguousarray(tag, dtype=np.float64), "ts": np.ascontiguousarray(ts, dtype=np.float64),
           "playtime": np.ascontiguousarray(playtime, dtype=np.float64),
           "duration": np.ascontiguousarray(duration, dtype=np.float64),
           "labels": np.ascontiguousarray(labels, dtype=np.uint32)}
    cont = np.ascontiguousarray(content, dtype=np.float64)
    seeds = np.ascontiguousarray(rng_seeds, dtype=np.uint64)
    sid_a = np.ascontiguousarray(sid, dtype=np.int32) if sid is not None else None
    P = C.POINTER
    rec = orx_records(off.ctypes.data_as(P(C.c_int64)), arr["vid"].ctypes.data_as(P(C.c_int64)),
                      arr["aid"].ctypes.data_as(P(C.c_int32)), arr["tag"].ctypes.data_as(P(C.c_double)),
                      arr["ts"].ctypes.data_as(P(C.c_double)), arr["playtime"].ctypes.data_as(P(C.c_double)),
                      arr["duration"].ctypes.data_as(P(C.c_double)), arr["labels"].ctypes.data_as(P(C.c_uint32)),
                      sid_a.ctypes.data_as(P(C.c_int32)) if sid_a is not None else None)
    out = {"offsets": np.empty(U + 1, dtype=np.int64), "vid": np.empty(n_out, dtype=np.int64),
           "aid": np.empty(n_out, dtype=np.int32), "tag": np.empty(n_out), "ts": np.empty(n_out),
           "playtime": np.empty(n_out), "duration": np.empty(n_out), "labels": np.empty(n_out, dtype=np.uint32)}
    if sid_a is not None:
        out["sid"] = np.empty(n_out * n_code_layers, dtype=np.int32)
    ro = orx_records_out(out["offsets"].ctypes.data_as(P(C.c_int64)), out["vid"].ctypes.data_as(P(C.c_int64)),
                         out["aid"].ctypes.data_as(P(C.c_int32)), out["tag"].ctypes.data_as(P(C.c_double)),
                         out["ts"].ctypes.data_as(P(C.c_double)), out["playtime"].ctypes.data_as(P(C.c_double)),
                         out["duration"].ctypes.data_as(P(C.c_double)), out["labels"].ctypes.data_as(P(C.c_uint32)),
                         out["sid"].ctypes.data_as(P(C.c_int32)) if sid_a is not None else None)
    check(lib().orx_compress_lifelong(device, U, C.byref(rec), cont.ctypes.data_as(P(C.c_double)),
                                      cont.shape[1] if cont.ndim == 2 else 1, threshold, max_out, n_code_layers,
                                      seeds.ctypes.data_as(P(C.c_uint64)), C.byref(ro)))
    return out

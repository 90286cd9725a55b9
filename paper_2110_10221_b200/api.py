"""Thin Python binding over the C ABI (include/cora.h).

PyTorch is used only for device memory (tensors as buffers) and streams; every step of the
path runs in the kernels of libcora_b200.so.  Function names follow the C entry points.
There is no CPU or eager fallback: a missing library or a non-CUDA tensor raises.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib as C

_ACT = {"none": C.CORA_ACT_NONE, None: C.CORA_ACT_NONE, "relu": C.CORA_ACT_RELU, "gelu": C.CORA_ACT_GELU_ERF}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("libcora_b200 takes contiguous CUDA tensors only (no CPU fallback)")


def _expect(t: Optional[torch.Tensor], shape, dtype, name: str, device=None, host: bool = False) -> None:
    """Size / dtype / device check before a raw pointer crosses the C ABI (an undersized buffer would be
    read or written out of range by the kernels or the copies)."""
    if t is None:
        return
    if host:
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name}: contiguous host tensor required (pinned for asynchronous copies)")
    elif not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: contiguous CUDA tensor required (no CPU fallback)")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")


class RaggedLayout:
    """Device offset tables of one ragged batch (cora_layout_build).  Reused across layers."""

    def __init__(self, lengths: torch.Tensor, total_tokens: int, heads: int, max_len: int, stream=None):
        _need_cuda(lengths)
        if lengths.dtype != torch.int32:
            raise ValueError("lengths must be int32")
        self.lengths = lengths
        B = lengths.numel()
        nbytes = C.lib().cora_layout_workspace_bytes(B, int(total_tokens), int(heads), int(max_len))
        if nbytes == 0:
            raise C.CoraError(C.CORA_ERR_INVALID, "cora_layout_workspace_bytes")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=lengths.device)
        self.c = C.Layout()
        C.check(C.lib().cora_layout_build(_ptr(lengths), B, int(total_tokens), int(heads), int(max_len), _ptr(self.ws),
                                          nbytes, ctypes.byref(self.c), _stream(stream)), "cora_layout_build")

    @property
    def batch(self):
        return self.c.batch

    @property
    def heads(self):
        return self.c.heads

    @property
    def total_tokens(self):
        return self.c.total_tokens

    def status(self, stream=None) -> int:
        """CORA_OK (0) or CORA_ERR_DATA (2); synchronises the stream."""
        return C.lib().cora_layout_status(ctypes.byref(self.c), _stream(stream))

    def _view(self, ptr: int, n: int, dtype) -> torch.Tensor:
        off = ptr - self.ws.data_ptr()
        size = torch.tensor([], dtype=dtype).element_size()
        return self.ws[off:off + n * size].view(dtype)

    def tables(self) -> dict:
        """Views of the device tables (for tests and inspection)."""
        B, T = self.c.batch, self.c.total_tokens
        return {
            "row_off": self._view(self.c.row_off, B + 1, torch.int32),
            "attn_off": self._view(self.c.attn_off, B + 1, torch.int64),
            "seq_of_tok": self._view(self.c.seq_of_tok, T, torch.int32),
            "pos_in_seq": self._view(self.c.pos_in_seq, T, torch.int32),
            "tiles": self._view(self.c.tiles, self.c.n_tiles_max, torch.int32),
            "tile_seq": self._view(self.c.tile_seq, 2 * self.c.n_tiles_max, torch.int32),
            "n_tiles": self._view(self.c.n_tiles, 1, torch.int32),
            "units": self._view(self.c.units, self.c.n_units_max, torch.int32),
            "unit_seq": self._view(self.c.unit_seq, 2 * self.c.n_units_max, torch.int32),
            "n_units": self._view(self.c.n_units, 1, torch.int32),
            "status": self._view(self.c.status, 1, torch.int32),
        }


def layout_build(lengths: torch.Tensor, total_tokens: int, heads: int, max_len: int = 512, stream=None) -> RaggedLayout:
    return RaggedLayout(lengths, total_tokens, heads, max_len, stream)


@dataclass
class EncoderParams:
    """Weights of one post-LN encoder layer (nn.Linear [out, in] bf16; LayerNorm fp32), on the GPU."""

    d_model: int
    heads: int
    d_ff: int
    w_qkv: torch.Tensor
    b_qkv: torch.Tensor
    w_o: torch.Tensor
    b_o: torch.Tensor
    ln1_g: torch.Tensor
    ln1_b: torch.Tensor
    w1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    b2: torch.Tensor
    ln2_g: torch.Tensor
    ln2_b: torch.Tensor
    ln_eps: float = 1e-5
    act: str = "relu"

    _names = ("w_qkv", "b_qkv", "w_o", "b_o", "ln1_g", "ln1_b", "w1", "b1", "w2", "b2", "ln2_g", "ln2_b")

    @classmethod
    def from_host(cls, w, device="cuda", act: str = "relu", ln_eps: float = 1e-5) -> "EncoderParams":
        """From an object with numpy attributes (e.g. synth.EncoderWeights)."""
        kw = {}
        for n in cls._names:
            dt = torch.float32 if n.startswith("ln") else torch.bfloat16
            kw[n] = torch.as_tensor(getattr(w, n)).to(dtype=dt).contiguous().to(device)
        return cls(w.d_model, w.heads, w.d_ff, act=act, ln_eps=ln_eps, **kw)

    def cstruct(self) -> C.EncoderParams:
        p = C.EncoderParams()
        p.d_model, p.heads, p.d_ff, p.ln_eps, p.act = self.d_model, self.heads, self.d_ff, self.ln_eps, _ACT[self.act]
        for n in self._names:
            t = getattr(self, n)
            _need_cuda(t)
            setattr(p, n, t.data_ptr())
        return p


class EncoderLayer:
    """Reusable encoder-layer call: caches the C parameter struct and the workspace."""

    def __init__(self, params: EncoderParams):
        self.params = params
        self.cp = params.cstruct()
        self.ws = None

    def workspace_bytes(self, total_tokens: int) -> int:
        return C.lib().cora_encoder_workspace_bytes(ctypes.byref(self.cp), int(total_tokens))

    def launches(self, total_tokens: int) -> int:
        """Kernels one layer call launches (5 with the fused GEMM + LayerNorm epilogues, else 7)."""
        return int(C.lib().cora_encoder_layer_launches(ctypes.byref(self.cp), int(total_tokens)))

    def __call__(self, x: torch.Tensor, layout: RaggedLayout, out: Optional[torch.Tensor] = None,
                 stream=None, events: Optional[Sequence["torch.cuda.Event"]] = None) -> torch.Tensor:
        """events: optional C.LAYER_EVENTS torch.cuda.Event objects recorded around every kernel."""
        T = layout.total_tokens
        _expect(x, (T, self.params.d_model), torch.bfloat16, "x")
        _expect(out, (T, self.params.d_model), torch.bfloat16, "out", x.device)
        nbytes = self.workspace_bytes(T)
        if self.ws is None or self.ws.numel() < nbytes or self.ws.device != x.device:
            self.ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=x.device)
        y = torch.empty_like(x) if out is None else out
        ev = None
        if events is not None:
            if len(events) != C.LAYER_EVENTS:
                raise ValueError(f"need {C.LAYER_EVENTS} events")
            for e in events:  # torch creates its CUDA events lazily, on first record
                if e.cuda_event == 0:
                    e.record(stream)
            ev = (ctypes.c_void_p * C.LAYER_EVENTS)(*[e.cuda_event for e in events])
        C.check(C.lib().cora_encoder_layer_fwd_ex(ctypes.byref(self.cp), ctypes.byref(layout.c), _ptr(x), _ptr(y),
                                                  _ptr(self.ws), self.ws.numel(), _stream(stream), ev),
                "cora_encoder_layer_fwd_ex")
        return y


class EncoderForward:
    """Lengths in, layer out (cora_encoder_forward): the prelude and the layer in one call; the QKV GEMM
    runs under the prelude.  `layout` (after a call) is the batch's layout, for status()."""

    def __init__(self, params: EncoderParams, max_len: int = 512):
        self.params = params
        self.cp = params.cstruct()
        self.max_len = int(max_len)
        self.ws = None
        self.layout = C.Layout()

    def __call__(self, lengths: torch.Tensor, total_tokens: int, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
        T, B = int(total_tokens), lengths.numel()
        _expect(lengths, (B,), torch.int32, "lengths")
        _expect(x, (T, self.params.d_model), torch.bfloat16, "x", lengths.device)
        _expect(out, (T, self.params.d_model), torch.bfloat16, "out", lengths.device)
        nbytes = int(C.lib().cora_encoder_forward_workspace_bytes(ctypes.byref(self.cp), B, T, self.max_len))
        if nbytes == 0:
            raise C.CoraError(C.CORA_ERR_INVALID, "cora_encoder_forward_workspace_bytes")
        if self.ws is None or self.ws.numel() < nbytes or self.ws.device != x.device:
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
        y = torch.empty_like(x) if out is None else out
        C.check(C.lib().cora_encoder_forward(ctypes.byref(self.cp), _ptr(lengths), B, T, self.max_len, _ptr(x), _ptr(y),
                                             _ptr(self.ws), self.ws.numel(), ctypes.byref(self.layout),
                                             _stream(stream)), "cora_encoder_forward")
        return y

    def status(self, stream=None) -> int:
        return C.lib().cora_layout_status(ctypes.byref(self.layout), _stream(stream))


class EncoderStack:
    """n encoder layers over one ragged batch sharing ONE layout (cora_encoder_stack_fwd): the prelude
    runs once per batch, the layers ping-pong between the output and a workspace buffer."""

    def __init__(self, params: Sequence[EncoderParams]):
        self.params = list(params)
        self.cps = (C.EncoderParams * len(self.params))(*[p.cstruct() for p in self.params])
        self.ws = None

    def __call__(self, x: torch.Tensor, layout: RaggedLayout, out: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
        T = layout.total_tokens
        _expect(x, (T, self.params[0].d_model), torch.bfloat16, "x")
        _expect(out, (T, self.params[0].d_model), torch.bfloat16, "out", x.device)
        n = len(self.params)
        nbytes = int(C.lib().cora_encoder_stack_workspace_bytes(self.cps, n, T))
        if self.ws is None or self.ws.numel() < nbytes or self.ws.device != x.device:
            self.ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=x.device)
        y = torch.empty_like(x) if out is None else out
        C.check(C.lib().cora_encoder_stack_fwd(self.cps, n, ctypes.byref(layout.c), _ptr(x), _ptr(y), _ptr(self.ws),
                                               self.ws.numel(), _stream(stream)), "cora_encoder_stack_fwd")
        return y


class HostForward:
    """End-to-end public call with HOST buffers (cora_encoder_forward_host): H2D of lengths and x,
    device prelude, the layer, D2H of y -- one C call, enqueued on the stream."""

    def __init__(self, params: EncoderParams, batch: int, total_tokens: int, max_len: int = 512, device="cuda"):
        self.params = params
        self.cp = params.cstruct()
        self.batch, self.total_tokens, self.max_len = int(batch), int(total_tokens), int(max_len)
        n = C.lib().cora_forward_host_workspace_bytes(ctypes.byref(self.cp), self.batch, self.total_tokens, self.max_len)
        if n == 0:
            raise C.CoraError(C.CORA_ERR_INVALID, "cora_forward_host_workspace_bytes")
        self.ws = torch.empty(n, dtype=torch.uint8, device=device)
        self.layout = C.Layout()

    def __call__(self, lengths_host: torch.Tensor, x_host: torch.Tensor, y_host: torch.Tensor, stream=None) -> None:
        d = self.params.d_model
        _expect(lengths_host, (self.batch,), torch.int32, "lengths_host", host=True)
        _expect(x_host, (self.total_tokens, d), torch.bfloat16, "x_host", host=True)
        _expect(y_host, (self.total_tokens, d), torch.bfloat16, "y_host", host=True)
        if int(lengths_host.sum()) != self.total_tokens:
            raise ValueError("sum(lengths_host) != total_tokens")
        C.check(C.lib().cora_encoder_forward_host(ctypes.byref(self.cp), _ptr(lengths_host), self.batch,
                                                  self.total_tokens, self.max_len, _ptr(x_host), _ptr(y_host),
                                                  _ptr(self.ws), self.ws.numel(), ctypes.byref(self.layout),
                                                  _stream(stream)), "cora_encoder_forward_host")

    def status(self, stream=None) -> int:
        return C.lib().cora_layout_status(ctypes.byref(self.layout), _stream(stream))


def encoder_layer(x: torch.Tensor, layout: RaggedLayout, params: EncoderParams, out=None, stream=None) -> torch.Tensor:
    return EncoderLayer(params)(x, layout, out=out, stream=stream)


def linear(a: torch.Tensor, w: torch.Tensor, bias: Optional[torch.Tensor] = None,
           residual: Optional[torch.Tensor] = None, act: str = "none", out=None, stream=None) -> torch.Tensor:
    m, k = a.shape
    n = w.shape[0]
    _expect(a, (m, k), torch.bfloat16, "a")
    _expect(w, (n, k), torch.bfloat16, "w", a.device)
    _expect(bias, (n,), torch.bfloat16, "bias", a.device)
    _expect(residual, (m, n), torch.bfloat16, "residual", a.device)
    _expect(out, (m, n), torch.bfloat16, "out", a.device)
    c = torch.empty(m, n, dtype=torch.bfloat16, device=a.device) if out is None else out
    C.check(C.lib().cora_linear_fwd(_ptr(a), _ptr(w), _ptr(bias), _ptr(residual), _ptr(c), m, n, k, _ACT[act],
                                    _stream(stream)), "cora_linear_fwd")
    return c


def linear_residual_layernorm(a: torch.Tensor, w: torch.Tensor, residual: torch.Tensor, gamma: torch.Tensor,
                              beta: torch.Tensor, bias: Optional[torch.Tensor] = None, eps: float = 1e-5,
                              act: str = "none", out=None, stream=None) -> torch.Tensor:
    """c = LN(act(a w^T + bias) + residual) with the LayerNorm fused into the GEMM epilogue (n == 512)."""
    m, k = a.shape
    n = w.shape[0]
    _expect(a, (m, k), torch.bfloat16, "a")
    _expect(w, (n, k), torch.bfloat16, "w", a.device)
    _expect(bias, (n,), torch.bfloat16, "bias", a.device)
    _expect(residual, (m, n), torch.bfloat16, "residual", a.device)
    _expect(gamma, (n,), torch.float32, "gamma", a.device)
    _expect(beta, (n,), torch.float32, "beta", a.device)
    _expect(out, (m, n), torch.bfloat16, "out", a.device)
    c = torch.empty(m, n, dtype=torch.bfloat16, device=a.device) if out is None else out
    C.check(C.lib().cora_linear_residual_layernorm_fwd(_ptr(a), _ptr(w), _ptr(bias), _ptr(residual), _ptr(gamma),
                                                       _ptr(beta), eps, _ptr(c), m, n, k, _ACT[act], _stream(stream)),
            "cora_linear_residual_layernorm_fwd")
    return c


class VgemmPlan:
    """The serialised vgemm work list (cora_vgemm_plan) in PINNED host memory, and its device workspace:
    reusable, and capturable in a CUDA graph (the plan copy is a memcpy node from pinned memory)."""

    def __init__(self, dims, m_max: int, n_max: int, k_max: int, device="cuda"):
        batch = len(dims)
        if any(len(row) != 3 for row in dims):
            raise ValueError("dims: [batch][3] (M_i, N_i, K_i)")
        self.dims = [tuple(int(v) for v in row) for row in dims]
        self.shape = (batch, int(m_max), int(n_max), int(k_max))
        dh = (ctypes.c_int32 * max(3 * batch, 1))(*[v for row in self.dims for v in row])
        n = int(C.lib().cora_vgemm_plan_bytes(batch, dh))
        if n == 0:
            raise C.CoraError(C.CORA_ERR_INVALID, "cora_vgemm_plan_bytes")
        self.host = torch.empty(n, dtype=torch.uint8).pin_memory()
        C.check(C.lib().cora_vgemm_plan(batch, dh, int(m_max), int(n_max), int(k_max), ctypes.c_void_p(self.host.data_ptr()),
                                        n), "cora_vgemm_plan")
        self.ws = torch.empty(max(n, 256), dtype=torch.uint8, device=device)


def vgemm(a: torch.Tensor, b: torch.Tensor, dims, out: Optional[torch.Tensor] = None, stream=None,
          plan: Optional[VgemmPlan] = None) -> torch.Tensor:
    """C_i = A_i B_i over padded buffers a [batch, M_max, K_max], b [batch, K_max, N_max] (bf16); dims:
    [batch][3] host ints (M_i, N_i, K_i) (or a prebuilt `plan`).  Returns c [batch, M_max, N_max]; only
    C_i[:M_i, :N_i] is written (the rest of `out` is left as it was; a fresh `out` is zero-filled)."""
    _need_cuda(a, b, out)
    batch, m_max, k_max = a.shape
    n_max = b.shape[2]
    if b.shape[:2] != (batch, k_max) or a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ValueError("a [batch, M_max, K_max], b [batch, K_max, N_max], bf16")
    if plan is None:
        if len(dims) != batch:
            raise ValueError("dims: [batch][3] (M_i, N_i, K_i)")
        plan = VgemmPlan(dims, m_max, n_max, k_max, device=a.device)
    elif plan.shape != (batch, m_max, n_max, k_max):
        raise ValueError("plan built for other buffer shapes")
    _expect(out, (batch, m_max, n_max), torch.bfloat16, "out", a.device)
    c = torch.zeros(batch, m_max, n_max, dtype=torch.bfloat16, device=a.device) if out is None else out
    C.check(C.lib().cora_vgemm_fwd(ctypes.c_void_p(plan.host.data_ptr()), _ptr(a), _ptr(b), _ptr(c), m_max, n_max, k_max,
                                   _ptr(plan.ws), plan.ws.numel(), _stream(stream)), "cora_vgemm_fwd")
    return c


def trmm(l: torch.Tensor, b: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """c = tril(l) b (bf16; l [n, n], b [n, n_cols]); only the lower triangle of l is read."""
    _need_cuda(l, b, out)
    n, n_cols = b.shape
    if l.shape != (n, n) or l.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ValueError("l [n, n], b [n, n_cols], bf16")
    _expect(out, (n, n_cols), torch.bfloat16, "out", b.device)
    c = torch.empty(n, n_cols, dtype=torch.bfloat16, device=b.device) if out is None else out
    C.check(C.lib().cora_trmm_fwd(_ptr(l), _ptr(b), _ptr(c), n, n_cols, _stream(stream)), "cora_trmm_fwd")
    return c


def ragged_attention(layout: RaggedLayout, qkv: torch.Tensor, head_dim: int, scale: Optional[float] = None,
                     out=None, stream=None, causal: bool = False) -> torch.Tensor:
    T = layout.total_tokens
    d = layout.heads * head_dim
    _expect(qkv, (T, 3 * d), torch.bfloat16, "qkv")
    _expect(out, (T, d), torch.bfloat16, "out", qkv.device)
    o = torch.empty(T, d, dtype=torch.bfloat16, device=qkv.device) if out is None else out
    s = head_dim ** -0.5 if scale is None else scale
    fn = C.lib().cora_ragged_masked_attention_fwd if causal else C.lib().cora_ragged_attention_fwd
    C.check(fn(ctypes.byref(layout.c), _ptr(qkv), _ptr(o), head_dim, s, _stream(stream)),
            "cora_ragged_masked_attention_fwd" if causal else "cora_ragged_attention_fwd")
    return o


def ragged_softmax(layout: RaggedLayout, x: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    if x.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("x: bf16 or fp32")
    if layout.c.total_attn < 0:
        layout.status()  # once per layout: fills layout.c.total_attn (the size check needs S2 on the host)
    n = layout.heads * int(layout.c.total_attn)
    _expect(x, (n,), x.dtype, "x")
    _expect(out, (n,), x.dtype, "out", x.device)
    dt = {torch.bfloat16: C.CORA_DT_BF16, torch.float32: C.CORA_DT_F32}[x.dtype]
    y = torch.empty_like(x) if out is None else out
    C.check(C.lib().cora_ragged_softmax_fwd(ctypes.byref(layout.c), _ptr(x), _ptr(y), dt, _stream(stream)),
            "cora_ragged_softmax_fwd")
    return y


def layernorm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, residual: Optional[torch.Tensor] = None,
              eps: float = 1e-5, out=None, stream=None) -> torch.Tensor:
    if x.dtype not in (torch.bfloat16, torch.float32) or x.dim() != 2:
        raise ValueError("x: bf16 or fp32 [rows, cols]")
    rows, cols = x.shape
    _expect(x, (rows, cols), x.dtype, "x")
    _expect(residual, (rows, cols), x.dtype, "residual", x.device)
    _expect(gamma, (cols,), torch.float32, "gamma", x.device)
    _expect(beta, (cols,), torch.float32, "beta", x.device)
    _expect(out, (rows, cols), x.dtype, "out", x.device)
    dt = {torch.bfloat16: C.CORA_DT_BF16, torch.float32: C.CORA_DT_F32}[x.dtype]
    y = torch.empty_like(x) if out is None else out
    C.check(C.lib().cora_layernorm_fwd(_ptr(x), _ptr(residual), _ptr(gamma), _ptr(beta), _ptr(y), rows, cols, eps, dt,
                                       _stream(stream)), "cora_layernorm_fwd")
    return y


def shard_plan(lengths: Sequence[int], d_model: int, d_ff: int, n_ranks: int, rows: bool = False):
    """cora_shard_plan: seq_begin[n_ranks + 1] (and row_begin[n_ranks + 1] with rows=True)."""
    B = len(lengths)
    arr = (ctypes.c_int32 * max(B, 1))(*[int(x) for x in lengths])
    out = (ctypes.c_int32 * (n_ranks + 1))()
    rb = (ctypes.c_int32 * (n_ranks + 1))()
    C.check(C.lib().cora_shard_plan(arr, B, d_model, d_ff, n_ranks, out, rb), "cora_shard_plan")
    return (list(out), list(rb)) if rows else list(out)


def shard_groups(lengths: Sequence[int], seq_begin: Sequence[int], n_groups: int):
    """cora_shard_groups: (group_seq, group_row), each [n_ranks][n_groups + 1] nested lists."""
    B, R = len(lengths), len(seq_begin) - 1
    arr = (ctypes.c_int32 * max(B, 1))(*[int(x) for x in lengths])
    sb = (ctypes.c_int32 * (R + 1))(*[int(x) for x in seq_begin])
    gs = (ctypes.c_int32 * (R * (n_groups + 1)))()
    gr = (ctypes.c_int32 * (R * (n_groups + 1)))()
    C.check(C.lib().cora_shard_groups(arr, B, sb, R, n_groups, gs, gr), "cora_shard_groups")
    g = n_groups + 1
    return [list(gs[r * g:(r + 1) * g]) for r in range(R)], [list(gr[r * g:(r + 1) * g]) for r in range(R)]


def build_info() -> str:
    return C.lib().cora_build_info().decode()

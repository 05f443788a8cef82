"""Encoder/decoder layer executor over the fused templates (the preset chains of
build_preset_graph, fusion.hpp:343-397), B200 fusion scheme:

  bert-layer (post-norm, GELU)            gpt-layer / t5-layer (pre-norm, GELU / ReLU)
  -------------------------------------   -------------------------------------------------
  qkv = X Wqkv + b            [tcgen05]   h   = LN1(X)                         [mi_chain]
  A   = MHA(q, k, v; mask)    [attention] qkv = h Wqkv + b                     [tcgen05]
  X1  = LN(A Wo + bo + X)     [tcgen05]   A   = MHA(q, k, v; mask)             [attention]
  F   = GELU(X1 W1 + b1)      [tcgen05]   X1  = A Wo + bo + X ; h2 = LN2(X1)   [tcgen05, 2 outs]
  Y   = LN(F W2 + b2 + X1)    [tcgen05]   F   = act(h2 W1 + b1)                [tcgen05]
                                          Y   = F W2 + b2 + X1                 [tcgen05]

`compat=True` reproduces the reference chain exactly as the reference executes it: no QKV
projection (Q = K = V = the MHA input, backend.hpp:345-346) and every residual Add adds its
recorded `aux` matrix (backend.hpp:98-100), so results can be compared with CpuBackend::run_chain.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Optional

import torch

from . import fused
from . import sparsefuse as sf


@dataclass
class LayerShape:
    bs: int
    seq_len: int
    hidden: int = 768
    heads: int = 12
    head_size: int = 64
    ff: int = 0

    def __post_init__(self):
        if self.ff == 0:
            self.ff = 4 * self.hidden  # GraphHyper ff_dim = 0 -> 4 * hidden (fusion.hpp:351)

    @property
    def rows(self):
        return self.bs * self.seq_len


def init_weights(model: str, s: LayerShape, dtype=torch.float16, device="cuda", seed: int = 1,
                 compat: bool = False) -> Dict[str, torch.Tensor]:
    """Random-init weights of the architecture (synthetic; no checkpoints offline). Gemm weights
    U(+-1/sqrt(inner)), bias U[-0.5,0.5), LN gamma U[0.5,1.5), beta U[-0.5,0.5) like GraphData."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    H, F = s.hidden, s.ff

    def w(n, k):
        a = 1.0 / k ** 0.5
        return ((torch.rand(n, k, generator=g) * 2 - 1) * a).to(device, dtype)

    def u(n, lo, hi):
        return (lo + torch.rand(n, generator=g) * (hi - lo)).to(device, torch.float32)

    W = {"wo": w(H, H), "bo": u(H, -0.5, 0.5), "w1": w(F, H), "b1": u(F, -0.5, 0.5), "w2": w(H, F),
         "b2": u(H, -0.5, 0.5), "ln1_g": u(H, 0.5, 1.5), "ln1_b": u(H, -0.5, 0.5), "ln2_g": u(H, 0.5, 1.5),
         "ln2_b": u(H, -0.5, 0.5)}
    if not compat:
        W["wqkv"] = w(3 * H, H)
        W["bqkv"] = u(3 * H, -0.5, 0.5)
    if model == "t5-decoder-layer":  # the cross-attention block (DecoderLayer)
        W.update({"wqc": w(H, H), "bqc": u(H, -0.5, 0.5), "wkvc": w(2 * H, H), "bkvc": u(2 * H, -0.5, 0.5),
                  "woc": w(H, H), "boc": u(H, -0.5, 0.5), "ln3_g": u(H, 0.5, 1.5), "ln3_b": u(H, -0.5, 0.5)})
    return W


class EncoderLayer:
    """One layer of `model` on a fixed (bs, seq_len) with activations resident in HBM."""

    def __init__(self, model: str, shape: LayerShape, weights: Dict[str, torch.Tensor], ctx: sf.MhaContext,
                 compat: bool = False, aux: Optional[Dict[str, torch.Tensor]] = None, dtype=torch.float16,
                 ln_split: bool = False):
        if model not in ("bert-layer", "gpt-layer", "t5-layer"):
            raise sf._lib.InvalidParameter(f"unknown preset model: {model}")  # fusion.hpp:394
        if shape.heads * shape.head_size != shape.hidden:
            raise sf._lib.ShapeError("activation shape incompatible with MHA reshape")  # backend.hpp:331
        if ctx.mask.seq_len != shape.seq_len:
            raise sf._lib.ShapeError("MHA mask seq_len mismatch")  # backend.hpp:333
        self.model, self.s, self.W, self.ctx, self.compat = model, shape, weights, ctx, compat
        # ln_split: residual+LayerNorm as a separate MiChain pass after the GEMM (+bias+residual)
        # instead of inside the GEMM epilogue (the fusion search's choice at the BASELINE shapes)
        self.ln_split = ln_split
        self.aux = aux or {}
        self.act = "relu" if model == "t5-layer" else "gelu"
        M, H, F = shape.rows, shape.hidden, shape.ff
        dev = weights["wo"].device
        e = lambda *sz: torch.empty(*sz, dtype=dtype, device=dev)
        self.qkv = None if compat else e(M, 3 * H)
        self.h = e(M, H)       # pre-norm LN1 output
        self.attn = e(M, H)
        self.x1 = e(M, H)
        self.h2 = e(M, H)
        self.f = e(M, F)
        self.out = e(M, H)
        self.tmp = e(M, H) if ln_split else None
        self.graph = None
        self.graph_timed = None
        self.marks = []

    # (bs, heads, seq, d) views of a (bs*seq, width) activation at column offset c0
    def _heads(self, t: torch.Tensor, c0: int) -> torch.Tensor:
        s = self.s
        return t[:, c0:c0 + s.hidden].view(s.bs, s.seq_len, s.heads, s.head_size).permute(0, 2, 1, 3)

    def _mha(self, src: torch.Tensor, stream=None, mark=None):
        H = self.s.hidden
        if self.compat:
            q = k = v = self._heads(src, 0)
        else:
            fused.gemm_fused(src, self.W["wqkv"], self.qkv, bias=self.W["bqkv"], stream=stream)
            mark("qkv_gemm")
            q, k, v = self._heads(self.qkv, 0), self._heads(self.qkv, H), self._heads(self.qkv, 2 * H)
        sf.mha(q, k, v, self.ctx, out=self._heads(self.attn, 0), stream=stream)
        mark("masked_mha")

    def forward(self, x: torch.Tensor, stream=None, mark=None) -> torch.Tensor:
        """One layer step. `mark(name)`, if given, is called after each launch (the bench records a
        timing event there)."""
        W, A = self.W, self.aux
        mark = mark or (lambda name: None)
        if self.model == "bert-layer":
            self._mha(x, stream, mark)
            self._gemm_ln(self.attn, "wo", "bo", A.get("add1", x), "ln1", self.x1, None, "out_proj", stream, mark)
            fused.gemm_fused(self.x1, W["w1"], self.f, bias=W["b1"], act="gelu", stream=stream)
            mark("ffn1_gemm_gelu")
            self._gemm_ln(self.f, "w2", "b2", A.get("add2", self.x1), "ln2", self.out, None, "ffn2", stream, mark)
        else:
            fused.mi_chain(x, self.h, ln_gamma=W["ln1_g"], ln_beta=W["ln1_b"], stream=stream)
            mark("ln1_mi_chain")
            self._mha(self.h, stream, mark)
            self._gemm_ln(self.attn, "wo", "bo", A.get("add1", x), "ln2", self.h2, self.x1, "out_proj", stream, mark)
            fused.gemm_fused(self.h2, W["w1"], self.f, bias=W["b1"], act=self.act, stream=stream)
            mark("ffn1_gemm_act")
            fused.gemm_fused(self.f, W["w2"], self.out, bias=W["b2"], aux=A.get("add2", self.x1), stream=stream)
            mark("ffn2_gemm")
        return self.out

    def _gemm_ln(self, x, w, b, aux, ln, out, pre, name, stream, mark):
        """out = LN(x @ W^T + bias + aux) (pre, if given, receives the pre-LN sum): fused into the
        GEMM epilogue (cluster LayerNorm), or GEMM(+bias+aux) followed by a MiChain LN pass."""
        W = self.W
        if not self.ln_split:
            fused.gemm_fused(x, W[w], out, bias=W[b], aux=aux, ln_gamma=W[ln + "_g"], ln_beta=W[ln + "_b"],
                             out_pre_ln=pre, stream=stream)
            mark(name + "_gemm_ln")
            return
        mid = pre if pre is not None else self.tmp
        fused.gemm_fused(x, W[w], mid, bias=W[b], aux=aux, stream=stream)
        mark(name + "_gemm")
        fused.mi_chain(mid, out, ln_gamma=W[ln + "_g"], ln_beta=W[ln + "_b"], stream=stream)
        mark(name + "_ln")

    def kernels_per_step(self) -> int:
        n = 4 if self.model == "bert-layer" else 5
        n += (2 if self.model == "bert-layer" else 1) if self.ln_split else 0
        return n + (0 if self.compat else 1)

    # CUDA graph of one step (launch-bound small configs). timed=True adds an event-record node
    # before the first launch and after every launch (self.marks: [(name, event)], "start" first),
    # so per-kernel device time is read from the real step without host overhead.
    def capture(self, x: torch.Tensor, timed: bool = False) -> None:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.forward(x, stream=s)  # warm (tensor maps, attributes)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        self.marks = []
        mark = None
        if timed:
            def mark(name):
                e = torch.cuda.Event(enable_timing=True, external=True)
                e.record(s)
                self.marks.append((name, e))
        with torch.cuda.graph(g, stream=s):
            if timed:
                mark("start")
            self.forward(x, stream=s, mark=mark)
        if timed:
            self.graph_timed = g
        else:
            self.graph = g

    def kernel_ms(self) -> Dict[str, float]:
        """Per-launch device time of the last replay of a timed capture."""
        return {n: a.elapsed_time(b) for (_, a), (n, b) in zip(self.marks, self.marks[1:])}

    def replay(self, timed: bool = False):
        (self.graph_timed if timed else self.graph).replay()
        return self.out


class DecoderLayer(EncoderLayer):
    """T5-style decoder layer (pre-norm, ReLU): masked self-attention, encoder-decoder
    cross-attention, feed-forward. The reference's t5-layer preset is the encoder block only
    (fusion.hpp:379-392; the reference has no cross-attention); this adds the cross-attention
    block between the self-attention and FFN blocks, built from the same templates:

      h   = LN1(X)                                  [mi_chain]
      qkv = h Wqkv + b                              [tcgen05]
      A   = MHA(q, k, v; self mask, e.g. causal)    [attention]
      X1  = A Wo + bo + X ;  h2 = LN2(X1)           [tcgen05, 2 outputs]
      qc  = h2 Wqc + bqc                            [tcgen05]
      kvc = E Wkvc + bkvc                           [tcgen05]   E: the encoder output
      C   = MHA(qc, kc, vc; cross mask)             [attention]
      X2  = C Woc + boc + X1 ;  h3 = LN3(X2)        [tcgen05, 2 outputs]
      F   = relu(h3 W1 + b1)                        [tcgen05]
      Y   = F W2 + b2 + X2                          [tcgen05]

    Decoder and encoder sequences have the same length (the reference's masks are square); the
    cross mask is any DenseMask of that length (all-ones for dense cross-attention)."""

    def __init__(self, shape: LayerShape, weights: Dict[str, torch.Tensor], self_ctx: sf.MhaContext,
                 cross_ctx: sf.MhaContext, dtype=torch.float16, ln_split: bool = False):
        super().__init__("t5-layer", shape, weights, self_ctx, dtype=dtype, ln_split=ln_split)
        if cross_ctx.mask.seq_len != shape.seq_len:
            raise sf._lib.ShapeError("MHA mask seq_len mismatch")  # backend.hpp:333
        self.model = "t5-decoder-layer"
        self.cross_ctx = cross_ctx
        M, H = shape.rows, shape.hidden
        dev = weights["wo"].device
        e = lambda *sz: torch.empty(*sz, dtype=dtype, device=dev)
        # cross q | k | v in one (M, 3H) buffer (the two projections write column slices), so the
        # three attention views share strides as the executor's argument block requires
        self.qkvc, self.cattn, self.x2, self.h3 = e(M, 3 * H), e(M, H), e(M, H), e(M, H)
        self.enc = None

    def forward(self, x: torch.Tensor, enc: Optional[torch.Tensor] = None, stream=None, mark=None) -> torch.Tensor:
        W = self.W
        mark = mark or (lambda name: None)
        enc = enc if enc is not None else self.enc
        if enc is None or enc.shape != x.shape:
            raise sf._lib.ShapeError("decoder layer needs the encoder output (bs*seq x hidden)")
        H = self.s.hidden
        fused.mi_chain(x, self.h, ln_gamma=W["ln1_g"], ln_beta=W["ln1_b"], stream=stream)
        mark("ln1_mi_chain")
        self._mha(self.h, stream, mark)
        self._gemm_ln(self.attn, "wo", "bo", x, "ln2", self.h2, self.x1, "out_proj", stream, mark)
        # cross-attention: queries from the decoder stream, keys / values from the encoder output
        fused.gemm_fused(self.h2, W["wqc"], self.qkvc[:, :H], bias=W["bqc"], stream=stream)
        mark("cross_q_gemm")
        fused.gemm_fused(enc, W["wkvc"], self.qkvc[:, H:], bias=W["bkvc"], stream=stream)
        mark("cross_kv_gemm")
        sf.mha(self._heads(self.qkvc, 0), self._heads(self.qkvc, H), self._heads(self.qkvc, 2 * H), self.cross_ctx,
               out=self._heads(self.cattn, 0), stream=stream)
        mark("cross_mha")
        self._gemm_ln(self.cattn, "woc", "boc", self.x1, "ln3", self.h3, self.x2, "cross_out", stream, mark)
        fused.gemm_fused(self.h3, W["w1"], self.f, bias=W["b1"], act="relu", stream=stream)
        mark("ffn1_gemm_act")
        fused.gemm_fused(self.f, W["w2"], self.out, bias=W["b2"], aux=self.x2, stream=stream)
        mark("ffn2_gemm")
        return self.out

    def kernels_per_step(self) -> int:
        return 10 + (2 if self.ln_split else 0)

    def capture(self, x: torch.Tensor, enc: Optional[torch.Tensor] = None, timed: bool = False) -> None:
        self.enc = enc if enc is not None else self.enc
        super().capture(x, timed)

"""Dense tower of the hybrid step.

The reference's NN worker trains a small feed-forward CTR net on the pooled embeddings
joined with the non-id features (``DenseNet`` dense_nn.hpp:37-199, ``NnWorker::
train_step`` nn_worker.hpp:461-487) and averages the dense gradient over the K
trainers with a synchronous all-reduce (``AllReduceHub`` nn_worker.hpp:73-244). Here
that tower runs on the GPU next to the embedding path:

* parameters live in ONE flat fp32 device vector with the reference's layout (per
  layer: W[out][in] row-major, then b[out]; dense_nn.hpp:45-52) and the reference's
  Glorot init drawn from ``Rng(mix64(init_seed))`` (nn_worker.hpp:335, dense_nn.hpp:
  55-65), so a checkpoint or a replica compares element for element;
* forward/backward are cuBLAS fp32 GEMMs (plain library GEMMs: no TF32, the reference
  computes in fp32) over the whole batch instead of per-sample loops, so results match
  the reference within fp32 summation-order tolerance, not bitwise;
* the dense-gradient all-reduce reproduces the reference's canonical mean BIT-EXACTLY
  (stride-doubling tree over ascending rank, then one division by K,
  nn_worker.hpp:214-226): a reduce-scatter by all-to-all (each rank receives every
  rank's slice of one chunk), the tree over ranks on that slice, an all-gather of the
  reduced slices -- the same bytes on the wire as a ring all-reduce;
* ``sgd_step`` refuses non-finite gradients (dense_nn.hpp:263-273) and applies
  ``p -= lr * g`` with both operations rounded separately.
"""
from __future__ import annotations

import math

import numpy as np

from . import workloads as W
from .hps import DivergenceError, PreconditionError

BCE_CLAMP = 1e-7  # kBceClamp dense_nn.hpp:30


def glorot_params(dims, init_seed: int) -> np.ndarray:
    """DenseNet(dims, Rng(mix64(init_seed))) parameters (dense_nn.hpp:42-66): weights of
    every layer drawn in order from one Rng stream as (float)(-lim + 2lim*u), biases 0."""
    dims = list(dims) + [1]
    total = sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(len(dims) - 1))
    out = np.zeros(total, np.float32)
    seed = W.mix64_int(init_seed)
    drawn, off = 0, 0
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        lim = math.sqrt(6.0 / float(fi + fo))
        u = W.uniform01(seed, fi * fo, drawn)
        # uniform(lo, hi) = lo + (hi - lo) * u, in double (core.hpp:63), then narrowed
        out[off:off + fi * fo] = ((-lim) + (lim - (-lim)) * u).astype(np.float32)
        drawn += fi * fo
        off += fi * fo + fo
    return out


class DenseTower:
    """The reference's DenseNet (ReLU hidden layers, one logistic output) on one GPU."""

    def __init__(self, input_dim: int, hidden=(64, 32), init_seed: int = 0, device=None,
                 params: np.ndarray | None = None):
        import torch

        if input_dim <= 0:
            raise PreconditionError("DenseNet: input width must be positive")
        self.torch = torch
        self.dims = [int(input_dim)] + [int(h) for h in hidden] + [1]
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        host = glorot_params(self.dims[:-1], init_seed) if params is None else \
            np.ascontiguousarray(params, np.float32)
        self.params = torch.from_numpy(host).to(self.device)
        self.grad = torch.zeros_like(self.params)
        self.W, self.b, self.gW, self.gb = [], [], [], []
        off = 0
        for l in range(len(self.dims) - 1):
            fi, fo = self.dims[l], self.dims[l + 1]
            self.W.append(self.params[off:off + fi * fo].view(fo, fi))
            self.gW.append(self.grad[off:off + fi * fo].view(fo, fi))
            off += fi * fo
            self.b.append(self.params[off:off + fo])
            self.gb.append(self.grad[off:off + fo])
            off += fo
        self.param_count = off
        self._ones = {}

    def forward_backward(self, x, labels, input_grad=None, input_cols: int | None = None):
        """batch_forward_backward (dense_nn.hpp:218-246): mean BCE loss of the batch.
        Fills self.grad (the mean-loss dense gradient, params layout) and returns
        (mean_loss [device scalar], probs [B], input_grad [B, input_cols]). The loss
        derivative at the logit is (p - y) / B; the clamp only binds where the loss
        saturates. ``input_cols`` limits the input gradient to the leading columns (the
        embedding slice: split_group_grads dense_nn.hpp:251-261 drops the non-id tail).

        ``x`` may be a list of column blocks ([pooled embeddings, non-id features]): the
        first layer then multiplies each block by its slice of W0 (no concatenated copy of
        the input), and its weight gradient is assembled from the blocks' products."""
        t = self.torch
        parts = list(x) if isinstance(x, (list, tuple)) else [x]
        B = parts[0].shape[0]
        if B == 0:
            raise PreconditionError("batch_forward_backward: empty batch")
        widths = [p_.shape[1] for p_ in parts]
        L = len(self.W)
        pre, acts = [], [None]
        # layer 0 over the column blocks
        z = t.addmm(self.b[0], parts[0], self.W[0][:, :widths[0]].t())
        c0 = widths[0]
        for p_, w_ in zip(parts[1:], widths[1:]):
            z.addmm_(p_, self.W[0][:, c0:c0 + w_].t())
            c0 += w_
        pre.append(z)
        h = t.relu(z) if L > 1 else z
        acts.append(h)
        for l in range(1, L):
            z = t.addmm(self.b[l], h, self.W[l].t())
            pre.append(z)
            h = t.relu(z) if l + 1 < L else z
            acts.append(h)
        logit = pre[-1][:, 0]
        prob = t.sigmoid(logit)
        p = prob.clamp(BCE_CLAMP, 1.0 - BCE_CLAMP)
        loss = -(labels * t.log(p) + (1.0 - labels) * t.log(1.0 - p))
        mean_loss = loss.sum() * (1.0 / B)
        delta = ((prob - labels) * (1.0 / B)).unsqueeze(1)
        for l in range(L - 1, -1, -1):
            if l == 0:
                if len(parts) == 1:
                    self._weight_grad(delta, parts[0], self.gW[0])
                else:
                    c0 = 0
                    for p_, w_ in zip(parts, widths):
                        blk = t.empty((delta.shape[1], w_), dtype=delta.dtype,
                                      device=delta.device)
                        self._weight_grad(delta, p_, blk)
                        self.gW[0][:, c0:c0 + w_].copy_(blk)
                        c0 += w_
            else:
                self._weight_grad(delta, acts[l], self.gW[l])
            t.sum(delta, 0, out=self.gb[l])
            if l == 0:
                cols = sum(widths) if input_cols is None else input_cols
                if input_grad is None:
                    input_grad = t.empty((B, cols), dtype=delta.dtype, device=delta.device)
                t.mm(delta, self.W[0][:, :cols], out=input_grad)
                break
            delta = t.mm(delta, self.W[l]).mul_(pre[l - 1] > 0)
        return mean_loss, prob, input_grad

    def _weight_grad(self, delta, a, out):
        """out = delta^T a, a reduction over the batch (K = B) into a small [out, in]
        matrix: a plain GEMM gets only a handful of output tiles (64 x 1677 -> 27 CTAs
        for 148 SMs), so the batch is split into chunks reduced as one batched GEMM and
        their partial products summed (split-K; fp32 throughout)."""
        t = self.torch
        B = delta.shape[0]
        c = 1
        for cand in (16, 8, 4, 2):
            if B % cand == 0 and B // cand >= 512:
                c = cand
                break
        if c == 1:
            t.mm(delta.t(), a, out=out)
            return
        part = t.bmm(delta.view(c, B // c, -1).transpose(1, 2), a.view(c, B // c, -1))
        # sum of the c partial products as a GEMM with a ones row (a strided reduction
        # over the leading dimension is slower)
        key = (c, part.dtype, part.device)
        ones = self._ones.get(key)
        if ones is None:
            ones = self._ones[key] = t.ones((1, c), dtype=part.dtype, device=part.device)
        if out.is_contiguous():
            t.mm(ones, part.view(c, -1), out=out.view(1, -1))
        else:
            out.copy_(t.mm(ones, part.view(c, -1)).view_as(out))

    def sgd_step(self, grad, lr: float, finite=None):
        """sgd_step (dense_nn.hpp:263-273): p -= lr * g (both ops rounded). Non-finite
        gradients raise DivergenceError and leave the parameters untouched; pass
        ``finite`` (a device bool) to defer that check to the caller."""
        t = self.torch
        ok = t.isfinite(grad).all() if finite is None else finite
        if finite is None and not bool(ok):
            raise DivergenceError("sgd_step: non-finite gradient")
        step = grad * lr
        if finite is not None:  # no host sync: a non-finite gradient applies nothing
            step = t.where(ok, step, t.zeros((), dtype=step.dtype, device=step.device))
        self.params.sub_(step)


def canonical_mean(parts):
    """AllReduceHub::canonical_mean (nn_worker.hpp:214-226) over parts[K, n] (a torch
    tensor): stride-doubling pairwise sums over ascending rank, then one division."""
    K = parts.shape[0]
    acc = parts.clone()
    stride = 1
    while stride < K:
        # for lo in 0, 2s, 4s, ... while lo + s < K: acc[lo] += acc[lo + s]
        acc[0:K - stride:2 * stride] += acc[stride:K:2 * stride]
        stride *= 2
    return acc[0] / float(K)


def allreduce_mean(grad, group=None):
    """The reference's synchronous dense all-reduce, bit-exact (canonical_mean), over
    torch.distributed. NCCL: all-to-all reduce-scatter of K slices, the rank-ordered tree
    on this rank's slice, all-gather of the reduced slices. Other backends (gloo, CPU
    tests): all-gather of whole vectors and the tree locally."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return grad / 1.0
    K = dist.get_world_size(group)
    n = grad.numel()
    if dist.get_backend(group) != "nccl":
        parts = [torch.empty_like(grad) for _ in range(K)]
        dist.all_gather(parts, grad.contiguous(), group=group)
        return canonical_mean(torch.stack(parts))
    c = (n + K - 1) // K
    send = torch.zeros(K * c, dtype=grad.dtype, device=grad.device)
    send[:n] = grad.reshape(-1)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)  # recv[k] = rank k's slice for this rank
    mine = canonical_mean(recv.view(K, c))
    out = torch.empty(K * c, dtype=grad.dtype, device=grad.device)
    dist.all_gather_into_tensor(out, mine, group=group)
    return out[:n].view_as(grad)

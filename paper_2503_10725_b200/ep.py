"""Expert-parallel (EP) MoE layer: experts sharded over the GPUs of one node.

SURVEY.md §8(e): rank r of P owns experts [r*E/P, (r+1)*E/P); tokens are
data-parallel.  Per layer call there is one exchange each way:

  dispatch  route (all E, on device) -> samoyeds_ep_plan -> samoyeds_ep_pack
            -> all_to_all_v of bf16 token rows + tags (local expert ids, gate
               weights); one copy of a token per destination rank
  compute   samoyeds_moe_experts on the received rows (the rank's experts)
  combine   all_to_all_v of the fp32 partial rows back -> samoyeds_ep_combine

All compute runs in libsamoyeds kernels; torch.distributed (NCCL over
NVLink/NVSwitch on the GPU box, gloo in the CPU tests) only moves the buffers.
The split sizes need one device->host read of the [P] send counts per call.
The phases are separate methods so a test can drive several ranks inside one
process with an in-process exchange (tests/test_gpu_ep.py).
"""
from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist

from . import api


class TorchExchange:
    """all_to_all_v through a torch.distributed process group."""

    def __init__(self, group=None):
        self.group = group

    def counts(self, send_counts: List[int], device) -> List[int]:
        world = len(send_counts)
        send = torch.tensor(send_counts, dtype=torch.int64, device=device)
        recv = torch.empty(world, dtype=torch.int64, device=device)
        dist.all_to_all_single(recv, send, group=self.group)
        return [int(v) for v in recv.cpu().tolist()]

    def rows(self, send: torch.Tensor, send_splits: List[int], recv_splits: List[int]) -> torch.Tensor:
        # move raw bytes (bf16 bit patterns are int16, which NCCL has no type for)
        raw = send.contiguous().view(torch.uint8).reshape(send.shape[0], -1)
        out = torch.empty(sum(recv_splits), raw.shape[1], dtype=torch.uint8, device=send.device)
        dist.all_to_all_single(out, raw, output_split_sizes=recv_splits, input_split_sizes=send_splits,
                               group=self.group)
        return out.view(send.dtype).reshape((sum(recv_splits),) + tuple(send.shape[1:]))


def pack_tags(tag_ids: torch.Tensor, tag_w: torch.Tensor) -> torch.Tensor:
    """[S x k] int32 ids + [S x k] fp32 weights -> one int32 [S x 2k] buffer."""
    return torch.cat([tag_ids, tag_w.view(torch.int32)], dim=1)


def unpack_tags(tags: torch.Tensor, k: int):
    return tags[:, :k].contiguous(), tags[:, k:].contiguous().view(torch.float32)


class EPMoELayer:
    """MoE layer with experts sharded over `world` ranks (this rank = `rank`)."""

    def __init__(self, cfg: api.MoEConfig, local_experts, rank: int, world: int, max_tokens: int, device=None,
                 exchange: Optional[TorchExchange] = None):
        if cfg.num_experts % world:
            raise ValueError("num_experts must be divisible by the EP world size")
        self.cfg, self.rank, self.world = cfg, rank, world
        self.e_local = cfg.num_experts // world
        if len(local_experts) != self.e_local:
            raise ValueError(f"rank {rank} needs {self.e_local} local experts")
        self.local_cfg = api.MoEConfig(self.e_local, cfg.top_k, cfg.hidden, cfg.ffn, 0, cfg.gating, cfg.fmt, cfg.gate_up)
        self.device = device or torch.device("cuda")
        # a rank can receive every token of every rank once
        self.experts = api.MoEExperts(self.local_cfg, local_experts, max_rows=max(1, max_tokens * world),
                                      device=self.device)
        self.exchange = exchange

    # ---- phase 1
    def dispatch(self, x: torch.Tensor, logits: torch.Tensor):
        k = self.cfg.top_k
        ids, w, *_ = api.route(logits, k, self.cfg.gating)
        counts, offsets, sel, tag_ids, tag_w = api.ep_plan(ids, w, self.cfg.num_experts, self.world)
        send_counts = [int(v) for v in counts.cpu().tolist()]          # one D2H read per call
        S = sum(send_counts)
        x_send = api.ep_pack(x, offsets, sel, S)
        tags = pack_tags(tag_ids[:S], tag_w[:S])
        return {"send_counts": send_counts, "offsets": offsets, "sel": sel, "x_send": x_send, "tags": tags}

    # ---- phase 2
    def compute(self, x_recv: torch.Tensor, tags_recv: torch.Tensor) -> torch.Tensor:
        keys, vals = unpack_tags(tags_recv, self.cfg.top_k)
        return self.experts(x_recv, keys, vals)

    # ---- phase 3
    def combine(self, back: torch.Tensor, state, out: torch.Tensor) -> torch.Tensor:
        out.zero_()
        return api.ep_combine(back, state["offsets"], state["sel"], out)

    def __call__(self, x: torch.Tensor, logits: torch.Tensor, out: Optional[torch.Tensor] = None):
        ex = self.exchange or TorchExchange()
        if out is None:
            out = torch.empty(x.shape[0], self.cfg.hidden, dtype=torch.float32, device=x.device)
        st = self.dispatch(x, logits)
        recv_counts = ex.counts(st["send_counts"], x.device)
        x_recv = ex.rows(st["x_send"], st["send_counts"], recv_counts)
        tags_recv = ex.rows(st["tags"], st["send_counts"], recv_counts)
        part = self.compute(x_recv, tags_recv)
        back = ex.rows(part, recv_counts, st["send_counts"])
        return self.combine(back, st, out)

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
        self.local_cfg = api.MoEConfig(self.e_local, cfg.top_k, cfg.hidden, cfg.ffn, 0, cfg.gating, cfg.fmt, cfg.gate_up,
                                       cfg.transcode)
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


# ------------------------------------------------ EP over NVLink peer memory

class SymmetricPeers:
    """Every rank's activations x [T_max x d] (bf16 bits) and fp32 output
    [T_max x d] in torch symmetric memory: each rank holds device pointers to
    all ranks' buffers (NVLink peer mappings), and a stream-ordered device
    barrier over the group."""

    def __init__(self, group, max_tokens: int, hidden: int, device):
        import torch.distributed._symmetric_memory as symm_mem
        self.x = symm_mem.empty(max_tokens, hidden, dtype=torch.int16, device=device)
        self.out = symm_mem.empty(max_tokens, hidden, dtype=torch.float32, device=device)
        self._hx = symm_mem.rendezvous(self.x, group)
        self._ho = symm_mem.rendezvous(self.out, group)
        self.x_ptrs = list(self._hx.buffer_ptrs)
        self.out_ptrs = list(self._ho.buffer_ptrs)

    def barrier(self):
        self._hx.barrier(channel=0)


class LocalPeers:
    """The same interface for `world` simulated ranks inside one process on one
    GPU (tests): plain device buffers, pointers valid on this device, and no
    barrier (the driver runs the phases of all ranks in order on one stream)."""

    def __init__(self, world: int, max_tokens: int, hidden: int, device):
        self.xs = [torch.zeros(max_tokens, hidden, dtype=torch.int16, device=device) for _ in range(world)]
        self.outs = [torch.zeros(max_tokens, hidden, dtype=torch.float32, device=device) for _ in range(world)]
        self.x_ptrs = [t.data_ptr() for t in self.xs]
        self.out_ptrs = [t.data_ptr() for t in self.outs]

    def view(self, rank: int):
        v = LocalPeers.__new__(LocalPeers)
        v.x, v.out, v.x_ptrs, v.out_ptrs = self.xs[rank], self.outs[rank], self.x_ptrs, self.out_ptrs
        v.barrier = lambda: None
        return v


class PeerEPMoELayer:
    """Expert-parallel MoE layer whose token rows and partial outputs move over
    NVLink peer memory INSIDE the SSMM kernels (include/samoyeds.h,
    samoyeds_moe_experts_peer): the owner's gate/up gathers each routed token
    straight from its source rank's x, its down scatter-adds straight into the
    source rank's output.  Per call only the routing metadata (row ids + tags,
    (1 + 2k) x 4 B per token and destination) crosses an all_to_all_v, plus
    two device barriers."""

    def __init__(self, cfg: api.MoEConfig, local_experts, rank: int, world: int, max_tokens: int, peers,
                 device=None, exchange: Optional[TorchExchange] = None):
        if cfg.num_experts % world:
            raise ValueError("num_experts must be divisible by the EP world size")
        if world > 8:
            raise ValueError("peer-memory EP spans one NVLink node (<= 8 ranks)")
        self.cfg, self.rank, self.world, self.peers = cfg, rank, world, peers
        self.e_local = cfg.num_experts // world
        if len(local_experts) != self.e_local:
            raise ValueError(f"rank {rank} needs {self.e_local} local experts")
        self.local_cfg = api.MoEConfig(self.e_local, cfg.top_k, cfg.hidden, cfg.ffn, 0, cfg.gating, cfg.fmt,
                                       cfg.gate_up, cfg.transcode)
        self.device = device or torch.device("cuda")
        self.max_tokens = max_tokens
        self.experts = api.MoEExperts(self.local_cfg, local_experts, max_rows=max(1, max_tokens * world),
                                      device=self.device)
        self.exchange = exchange

    # ---- phase 1: publish x, zero out, plan + row ids + tags
    def dispatch(self, x: torch.Tensor, logits: torch.Tensor):
        k = self.cfg.top_k
        T = x.shape[0]
        if T > self.max_tokens:
            raise ValueError("T exceeds max_tokens")
        xb = x.view(torch.int16) if x.dtype == torch.bfloat16 else x
        if xb.data_ptr() != self.peers.x.data_ptr():
            self.peers.x[:T].copy_(xb)
        self.peers.out[:T].zero_()
        ids, w, *_ = api.route(logits, k, self.cfg.gating)
        counts, offsets, sel, tag_ids, tag_w = api.ep_plan(ids, w, self.cfg.num_experts, self.world)
        send_counts = [int(v) for v in counts.cpu().tolist()]          # one D2H read per call
        S = sum(send_counts)
        row_ids = api.ep_row_ids(sel, offsets, self.rank, S)
        tags = torch.cat([row_ids[:S, None], tag_ids[:S], tag_w[:S].view(torch.int32)], dim=1)
        return {"send_counts": send_counts, "tags": tags, "T": T}

    # ---- phase 2: the rank's experts over the received rows, reading/adding peer memory
    def compute(self, tags_recv: torch.Tensor):
        k = self.cfg.top_k
        row_map = tags_recv[:, 0].contiguous()
        keys = tags_recv[:, 1:1 + k].contiguous()
        vals = tags_recv[:, 1 + k:].contiguous().view(torch.float32)
        self.experts.peer(self.world, self.peers.x_ptrs, self.cfg.hidden, self.peers.out_ptrs, self.cfg.hidden,
                          row_map, keys, vals)

    def __call__(self, x: torch.Tensor, logits: torch.Tensor, out: Optional[torch.Tensor] = None):
        ex = self.exchange or TorchExchange()
        st = self.dispatch(x, logits)
        recv_counts = ex.counts(st["send_counts"], x.device)
        tags_recv = ex.rows(st["tags"], st["send_counts"], recv_counts)
        self.peers.barrier()          # every rank's x published and output zeroed
        self.compute(tags_recv)
        self.peers.barrier()          # every owner's reductions into this rank's output done
        res = self.peers.out[:st["T"]]
        if out is None:
            return res.clone()
        return out.copy_(res)

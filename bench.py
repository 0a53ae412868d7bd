#!/usr/bin/env python
"""Benchmark: Samoyeds MoE layer on B200 (BASELINE.json metric:
"SSMM TFLOPS vs B200 2:4-sparse peak; MoE-layer tokens/s at 1/2/4/8 B200").

One step = one call of samoyeds_moe_layer (route + compaction, gate/up SSMM with
fused SiLU*up, down SSMM with fused routing-weight scale + scatter-add) over one
batch of T synthetic tokens per GPU, on a random-init layer of the named shape
in the (1,2,32) format (75% weight sparsity).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model mixtral|deepseek|qwen2] [--tokens T]

N > 1: one process per GPU (launched by torchrun, or spawned here when
WORLD_SIZE is unset); every rank runs its own batch of T tokens ("scaling":
"weak") through the expert-parallel layer -- experts sharded over the ranks,
token dispatch / combine over NCCL (default) or NVLink peer memory.  Rank 0
prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODELS = {
    # name: (hidden, ffn, experts, top_k, gating)
    "mixtral": (4096, 14336, 8, 2, "renorm_topk"),
    "deepseek": (2048, 1408, 64, 6, "softmax_all"),
    "qwen2": (3584, 2560, 64, 8, "softmax_all"),
}
WORKLOAD = {
    "mixtral": "mixtral-8x7b-moe-layer",
    "deepseek": "deepseek-moe-16b-moe-layer",
    "qwen2": "qwen2-57b-a14b-moe-layer",
}
FMT = (1, 2, 32)
BYTES_PER_ELEM = 0.578125     # canonical (1,2,32) bf16 weight bytes per logical element


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.4)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [ln for ts, ln in self.lines if t0 - 0.05 <= ts <= t1 + 0.05] or [ln for _, ln in self.lines[-3:]]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in rows:
            parts = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle

def oracle_sample(model: str, tokens: int, f_slice: int, rank: int = 0):
    """A bounded sample of the same workload for the CPU oracle: the first
    `tokens` tokens, all experts, and the first `f_slice` FFN channels of every
    expert (gate/up rows and down columns [0, f_slice)).  The FFN is a sum over
    its channels, so oracle time scales linearly with f: full-layer tokens/s =
    sample tokens/s * f_slice / ffn."""
    import numpy as np

    import synth
    from oracle import fmt as F
    d, f, E, k, gating = MODELS[model]
    fmt = F.SparseFormat(*FMT)
    experts = []
    for e in range(E):
        trip = []
        for i in range(3):
            if i < 2:   # gate/up rows [0, f_slice) of [f x d]
                w = synth.weight_bf16(synth.weight_seed(e, i), f, d, row_idx=np.arange(f_slice))
            else:       # down columns [0, f_slice) of [d x f]
                idx = (np.arange(d, dtype=np.uint64)[:, None] * np.uint64(f)
                       + np.arange(f_slice, dtype=np.uint64)[None, :])
                v = synth.fill_f32(synth.weight_seed(e, i), idx, synth.DIST_UNIFORM,
                                   synth.uniform_scale(np.sqrt(3.0 / f)))
                w = synth.f32_to_bf16_bits(v)
            trip.append(F.encode(F.prune(w, fmt), fmt))
        experts.append(tuple(trip))
    x = synth.activations_bf16(synth.SEED_X + 100 * rank, tokens, d)
    lg = synth.router_logits(synth.SEED_LOGITS + 100 * rank, tokens, E)
    return experts, x, lg, (0 if gating == "renorm_topk" else 1)


def time_oracle(model, tokens, f_slice, reps=1):
    from oracle import moe
    experts, x, lg, mode = oracle_sample(model, tokens, f_slice)
    d, f, E, k, _ = MODELS[model]
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        moe.moe_layer(experts, x, lg, k, mode)
        times.append(time.perf_counter() - t0)
    return times


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(model, tokens=128, f_slice=512):
    d, f, E, k, _ = MODELS[model]
    t = time_oracle(model, tokens, f_slice)[0]
    return {"value": tokens / t * f_slice / f, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
            "sample": f"{model} layer, {tokens} tokens, all {E} experts, FFN channels [0,{f_slice}) of {f} "
                      f"(time x {f}/{f_slice}); oracle fp64 NumPy; {t:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_cores()))
    model = args.model
    d, f, E, k, _ = MODELS[model]
    tokens, f_slice = 32, 128
    from oracle import moe
    experts, x, lg, mode = oracle_sample(model, tokens, f_slice)
    for _ in range(args.warmup):
        moe.moe_layer(experts, x, lg, k, mode)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        moe.moe_layer(experts, x, lg, k, mode)
    dt = (time.perf_counter() - t0) / args.steps
    value = tokens / dt * f_slice / f
    line = {"impl": "reference", "metric": "moe_layer_tokens_per_s", "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[model], "tokens_per_gpu": args.tokens, "format": "(1,2,32)",
                       "sample_tokens": tokens, "sample_ffn_channels": f_slice},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": f"each step: {tokens} tokens, {E} experts, FFN channels [0,{f_slice}) "
                                       f"of {f}, scaled x {f}/{f_slice}"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def build_layer(P, model, device, experts=None, transcode="auto", gate_up="auto"):
    import numpy as np
    import torch

    import synth
    d, f, E, k, gating = MODELS[model]
    fmt = P.Format(*FMT)
    experts_out = []
    for e in (range(E) if experts is None else experts):
        trip = []
        for i in range(3):
            rows, cols = (f, d) if i < 2 else (d, f)
            dense = torch.empty(rows, cols, dtype=torch.int16, device=device)
            P.synth_fill(dense, synth.weight_seed(e, i), synth.DIST_UNIFORM,
                         float(synth.uniform_scale(np.sqrt(3.0 / cols))))
            sw, status = P.compress(dense, fmt, prune=True)
            del dense
            trip.append(sw)
        experts_out.append(tuple(trip))
    # the layout the layer runs on (interleaved gate/up, one image block), then
    # drop everything the kernels do not read
    experts_out = P.prepare_experts(P.MoEConfig(E, k, d, f, 0, gating, fmt, gate_up, transcode), experts_out)
    for trip in experts_out:
        for sw in trip:
            if sw is not None:
                sw.drop_canonical()
    torch.cuda.synchronize()
    return experts_out


def free_port() -> int:
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-launch this command as N
    ranks of one node through torch.distributed.run (one process per GPU,
    rendezvous on 127.0.0.1); rank 0's JSON line comes back on stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def init_ranks(args, device=None):
    """The process group of an N-rank run (torchrun environment).  The rank count
    must equal --gpus.  NCCL's INFO log (communicator ranks: "nranks N") goes to
    stderr, so stdout keeps only the JSON line."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 or args.force_ep:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        backend = "gloo" if args.dry_run else "nccl"
        with stdout_to_stderr():     # NCCL's version banner goes to fd 1: keep stdout to the JSON line
            if backend == "nccl":
                dist.init_process_group(backend, rank=rank, world_size=world, device_id=device)
            else:
                dist.init_process_group(backend, rank=rank, world_size=world)
            dist.barrier()
        print(f"[bench] rank {rank}: process group backend={backend} nranks={dist.get_world_size()}",
              file=sys.stderr, flush=True)
    return world, rank


def run_dry(args):
    """--dry-run: the N-rank launch path without a GPU (gloo): every rank joins the
    process group, runs the barrier + max-over-ranks timing of the contract on a
    stand-in step, and rank 0 prints the contract line ("dry_run": true, no
    measurement).  Used by the CPU tests of the multi-GPU launcher."""
    import torch
    import torch.distributed as dist
    world, rank = init_ranks(args)
    d, f, E, k, gating = MODELS[args.model]
    t0 = time.perf_counter()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3])
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": "moe_layer_tokens_per_s", "value": None, "unit": "tokens/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                          "data": "synthetic", "dry_run": True,
                          "config": {"workload": WORKLOAD[args.model], "tokens_per_gpu": args.tokens,
                                     "global_tokens": args.tokens * world, "experts": E, "top_k": k,
                                     "parallelism": f"ep{world}" if world > 1 else "dp1"},
                          "barrier_ms_max_over_ranks": float(ms.item())}), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2503_10725_b200 as P

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    world, rank = init_ranks(args, device)
    lib = P.load()
    model = args.model
    d, f, E, k, gating = MODELS[model]
    T = args.tokens
    ep = (world > 1 or args.force_ep) and args.parallel == "ep"
    NS = args.shared
    if NS and (world > 1 or args.force_ep) and args.parallel == "ep":
        raise SystemExit("--shared: shared experts are measured on the 1-GPU / data-parallel layer")
    SG = args.shared_gate
    if SG == "sigmoid" and not NS:
        raise SystemExit("--shared-gate sigmoid needs --shared N")
    cfg = P.MoEConfig(E, k, d, f, NS, gating, P.Format(*FMT), args.gate_up, args.transcode, shared_gate=SG)
    transport = None
    comm = None
    x = torch.empty(T, d, dtype=torch.int16, device=device)
    if ep:
        from paper_2503_10725_b200.ep import EPMoELayer, PeerEPMoELayer, SymmetricPeers, TorchExchange
        if E % world:
            raise SystemExit(f"--parallel ep needs world | num_experts ({E})")
        el = E // world
        experts = build_layer(P, model, device, experts=range(rank * el, (rank + 1) * el), transcode=args.transcode)
        peers = None
        if args.ep_transport == "peer":
            try:      # token rows / outputs over NVLink peer memory inside the SSMM kernels
                with stdout_to_stderr():
                    peers = SymmetricPeers(dist.group.WORLD, T, d, device)
            except Exception as exc:  # no symmetric memory on this box: the NCCL transport
                print(f"symmetric memory unavailable ({exc}); using the NCCL transport", file=sys.stderr)
        if peers is not None:
            transport = "peer"
            layer = PeerEPMoELayer(cfg, experts, rank, world, T, peers, device=device, exchange=TorchExchange())
            x = peers.x[:T]               # inputs live in the symmetric buffer (no publish copy)
        elif args.ep_transport == "torch":
            transport = "torch"
            layer = EPMoELayer(cfg, experts, rank, world, max_tokens=T, device=device, exchange=TorchExchange())
        else:
            # default: the library's own NCCL communicator behind samoyeds_moe_layer(..., comm)
            # -- route, plan, grouped ncclSend/Recv of rows + tags, experts, fp32 partial
            # rows back, combine, all inside the C call (one host read of the counts)
            transport = "nccl"
            with stdout_to_stderr():
                comm = P.EPComm()
            print(f"[bench] rank {rank}: samoyeds EP communicator nranks={comm.world}", file=sys.stderr, flush=True)
            layer = P.MoELayer(cfg, experts, max_tokens=T, device=device, comm=comm)
    else:
        experts = build_layer(P, model, device, transcode=args.transcode, gate_up=args.gate_up)
        # shared experts: every token, weight 1 (reading R15);
        # weights drawn like routed experts E, E+1, ...
        shared = (build_layer(P, model, device, experts=range(E, E + NS), transcode=args.transcode, gate_up=args.gate_up)
                  if NS else ())
        layer = P.MoELayer(cfg, experts, shared=shared, max_tokens=T, device=device)

    P.synth_fill(x, synth.SEED_X + 100 * rank, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    lg = torch.empty(T, E + (NS if SG == "sigmoid" else 0), dtype=torch.float32, device=device)
    P.synth_fill(lg, synth.SEED_LOGITS + 100 * rank, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    if SG == "sigmoid":
        # one shared-expert gate logit per token (Qwen2-MoE: shared_expert_gate is Linear(d, 1)),
        # replicated into the columns of the NS width-f pieces of the wide shared FFN
        lg[:, E:] = lg[:, E:E + 1]
    out = torch.empty(T, d, dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- warm-up
    for _ in range(args.warmup):
        layer(x, lg, out)
    torch.cuda.synchronize()

    # ---------------- timed region (inputs resident in HBM)
    K = args.steps
    phase = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(K)]
    for evs in phase:           # torch creates the cudaEvent_t lazily on first record
        for ev in evs:
            ev.record(stream)
    torch.cuda.synchronize()
    handles = [(C_void_p_array(ev)) for ev in phase]
    # One layer call per step, each recording its phase events.  Single-GPU runs
    # capture the K calls into one CUDA graph (the layer never syncs with the
    # host) and replay it as the timed region: identical kernels, no launch gaps.
    use_graph = not args.no_graph and not ep

    def make_runner(xx, lgg, oo, hs, n):
        # hs: per-step phase-event arrays, or None for the clean steps that are timed
        # (each event-record node costs ~2.7 us inside the graph -- the empty
        # "zero_out" interval measures it -- so step times come from clean replays)
        def eager():
            for i in range(n):
                lib.smy_moe_set_phase_events(hs[i] if hs is not None else None, 6 if hs is not None else 0)
                layer(xx, lgg, oo)
            lib.smy_moe_set_phase_events(None, 0)
        if not use_graph:
            return eager, None
        g = torch.cuda.CUDAGraph()
        l0 = lib.smy_launch_count()
        with torch.cuda.graph(g):
            eager()
        n = lib.smy_launch_count() - l0
        g.replay()                       # warm replay
        torch.cuda.synchronize()
        return g.replay, n

    run, graph_launches = make_runner(x, lg, out, None, K)
    run_ph, _ = make_runner(x, lg, out, handles, K)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    launches0 = lib.smy_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.time()
    ev0.record(stream)
    run()
    ev1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    barrier()
    launches = graph_launches if graph_launches is not None else lib.smy_launch_count() - launches0
    clk = clocks.stop(t_wall0, t_wall1)
    ms = ev0.elapsed_time(ev1) / K
    # per-phase times (the roofline's kernel time): a second replay of the same steps
    # recording the layer's phase events; outside the timed region
    run_ph()
    torch.cuda.synchronize()
    ph = np.array([[phase[s][i].elapsed_time(phase[s][i + 1]) for i in range(5)] for s in range(K)])
    ph_ms = ph.mean(0)
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---------------- decode point on the same layer (reported beside the headline)
    dec = None
    if args.decode_tokens and args.decode_tokens < T and not ep:
        Td = args.decode_tokens
        xd, lgd, outd = x[:Td], lg[:Td], out[:Td]
        for _ in range(5):
            layer(xd, lgd, outd)
        torch.cuda.synchronize()
        Kd = max(20, K)
        dph = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(Kd)]
        for evs in dph:
            for ev in evs:
                ev.record(stream)
        torch.cuda.synchronize()
        dh = [C_void_p_array(ev) for ev in dph]
        drun, _ = make_runner(xd, lgd, outd, None, Kd)
        drun_ph, _ = make_runner(xd, lgd, outd, dh, Kd)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        drun()
        d1.record(stream)
        torch.cuda.synchronize()
        dms = d0.elapsed_time(d1) / Kd
        drun_ph()
        torch.cuda.synchronize()
        dpm = np.array([[dph[s][i].elapsed_time(dph[s][i + 1]) for i in range(5)] for s in range(Kd)]).mean(0)
        ids_d = P.route(lgd[:, :E].contiguous(), k, gating)[0].flatten().long()
        act_d = int((torch.bincount(ids_d, minlength=E) > 0).sum().item()) + NS   # + shared experts
        kd = k + NS                                   # rows per token through the grouped launches
        gu_bytes = 2 * act_d * f * d * BYTES_PER_ELEM + Td * kd * d * 2 + Td * kd * 4 + Td * kd * f * 2
        dn_bytes = act_d * f * d * BYTES_PER_ELEM + Td * kd * f * 2 + Td * kd * 8 + Td * kd * d * 4
        hbm_, _, _, _ = peaks()
        dec = {"tokens_per_gpu": Td, "tokens_per_s": Td * world / (dms * 1e-3), "ms_per_step": dms,
               "phases_ms": {"route_compact": dpm[0], "zero_out": dpm[1], "gate_up_ssmm": dpm[2], "down_ssmm": dpm[3]},
               "gate_up_hbm_frac": gu_bytes / (dpm[2] * 1e-3) / 1e9 / hbm_,
               "down_hbm_frac": dn_bytes / (dpm[3] * 1e-3) / 1e9 / hbm_,
               "layer_hbm_frac": (gu_bytes + dn_bytes) / (dms * 1e-3) / 1e9 / hbm_}

    # ---------------- end to end through the public call, from pinned host memory:
    # every step uploads its x + logits and downloads its fp32 output inside the
    # timed region; as in a serving loop, step s+1's upload and step s-1's
    # download run on copy streams beside step s's compute (double-buffered
    # device tensors, event-ordered), so e2e = max(PCIe, compute) when they overlap.
    # The single-GPU layer returns bf16 here (cfg.out_dtype = "bf16": fp32 accumulation,
    # one rounding -- what the next layer of a model consumes), halving the PCIe
    # download; the expert-parallel layer returns fp32.
    nb = 2
    e2e_bf16 = not ep and not args.e2e_f32
    e_layer = (P.MoELayer(P.MoEConfig(E, k, d, f, NS, gating, P.Format(*FMT), args.gate_up, args.transcode, "bf16",
                                      SG),
                          layer.experts, shared=layer.shared, max_tokens=T, device=device) if e2e_bf16 else layer)
    out_dt = torch.bfloat16 if e2e_bf16 else torch.float32
    x_h = x.cpu().pin_memory()
    lg_h = lg.cpu().pin_memory()
    out_h = [torch.empty(T, d, dtype=out_dt).pin_memory() for _ in range(nb)]
    xs = [x] + [torch.empty_like(x) for _ in range(nb - 1)]
    lgs = [lg] + [torch.empty_like(lg) for _ in range(nb - 1)]
    outs = [torch.empty(T, d, dtype=out_dt, device=device) for _ in range(nb)]
    h2d, d2h = torch.cuda.Stream(device), torch.cuda.Stream(device)
    ev_in = [torch.cuda.Event() for _ in range(nb)]
    ev_done = [torch.cuda.Event() for _ in range(nb)]
    ev_free = [torch.cuda.Event() for _ in range(nb)]

    def e2e_step(s_):
        i = s_ % nb
        with torch.cuda.stream(h2d):
            if s_ >= nb:
                h2d.wait_event(ev_done[i])        # step s-nb no longer reads xs[i] / lgs[i]
            xs[i].copy_(x_h, non_blocking=True)
            lgs[i].copy_(lg_h, non_blocking=True)
            ev_in[i].record(h2d)
        stream.wait_event(ev_in[i])
        if s_ >= nb:
            stream.wait_event(ev_free[i])         # step s-nb's output has been downloaded
        e_layer(xs[i], lgs[i], outs[i])
        ev_done[i].record(stream)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev_done[i])
            out_h[i].copy_(outs[i], non_blocking=True)
            ev_free[i].record(d2h)

    for s_ in range(max(2, args.warmup // 2) * nb):
        e2e_step(s_)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h2d.wait_stream(stream)
    for s_ in range(K):
        e2e_step(s_)
    stream.wait_stream(d2h)                       # the last download is inside the region
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = e0.elapsed_time(e1) / K
    if world > 1:
        t = torch.tensor([ms_e2e], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())

    # ---------------- roofline of the dominant kernel (gate/up SSMM)
    hbm, bf16_burst, bf16_sust, src = peaks()
    # the guide's rule: the burst dense figure for a kernel timed alone, the sustained
    # one (seconds back to back under the 1000 W cap) for a kernel timed inside a long
    # step loop -- which is what this timed region is whenever the clock sampler saw
    # sw_power_cap active in it; 2:4 sparse bf16 = 2 x dense (nominal ratio)
    capped = "sw_power_cap" in (clk.get("reasons") or []) and bf16_sust is not None
    dense_peak = bf16_sust if capped else bf16_burst
    sparse_peak = 2.0 * dense_peak
    cnt = torch.bincount(P.route(lg[:, :E].contiguous(), k, gating)[0].flatten().long(), minlength=E)
    if world > 1:
        dist.all_reduce(cnt)                 # assignments per expert over all ranks
    cnt = cnt.cpu().numpy()
    if ep:                                   # this rank computes its own experts for every rank's tokens
        el = E // world
        cnt = cnt[rank * el:(rank + 1) * el]
    else:
        cnt = cnt // max(world, 1) if world > 1 else cnt
    Tk = int(cnt.sum()) + NS * T             # (token, expert) pairs this GPU's gate/up SSMM processed
    #                                          (shared experts run as groups of the same launches)
    flops_gu = 2 * 2 * (f // 2) * d * Tk     # 2 weights x 2 * (f*N/M) * d * tokens
    active = int((cnt > 0).sum()) + NS
    bytes_gu = (2 * active * f * d * BYTES_PER_ELEM + Tk * d * 2 + Tk * 4 + Tk * f * 2)
    t_gu = ph_ms[2] * 1e-3
    ach_tf = flops_gu / t_gu / 1e12
    ach_gbs = bytes_gu / t_gu / 1e9
    ridge = sparse_peak * 1e12 / (hbm * 1e9)
    tensor_bound = flops_gu / bytes_gu >= ridge
    roof = ({"bound": "tensor", "achieved": ach_tf, "peak": sparse_peak, "unit": "TFLOP/s",
             "frac": ach_tf / sparse_peak, "traffic": None,
             "peak_source": (f"2 x {src} bf16 dense sustained ({bf16_sust} TF/s; timed region under sw_power_cap)"
                             if capped else f"2 x {src} bf16 dense burst ({bf16_burst} TF/s)"),
             "frac_of_burst": ach_tf / (2.0 * bf16_burst)} if tensor_bound else
            {"bound": "hbm", "achieved": ach_gbs, "peak": hbm, "unit": "GB/s", "frac": ach_gbs / hbm,
             "traffic": None, "peak_source": f"{src} hbm_gbs"})
    # the kernel the library launched (its own tile / CTA-pair decisions); under EP
    # the local experts' launch is approximated by the same rule on T*k/E rows each
    gu_name = (layer.kernel_names(T)[0] if isinstance(layer, P.MoELayer) and layer.comm is None
               else gate_up_kernel(T * k // E, f))
    roof["traffic"], roof["traffic_source"] = ncu_traffic(model, T, gu_name, NS)
    roof.update({"kernel": gu_name + " interleaved gate/up (fused SiLU*up)",
                 "per_launch_ms": ph_ms[2],
                 "algorithmic_flops": flops_gu, "algorithmic_bytes": bytes_gu,
                 "other_view": ({"achieved_gbs": ach_gbs, "hbm_frac": ach_gbs / hbm} if tensor_bound else
                                {"achieved_tflops": ach_tf, "sparse_frac": ach_tf / sparse_peak})})
    flops_layer = 3 * flops_gu / 2
    line = {
        "metric": "moe_layer_tokens_per_s", "value": T * world / (ms * 1e-3), "unit": "tokens/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": WORKLOAD[model] + (f"+{NS}shared" if NS else "") + ("-sigmoid-gated" if SG == "sigmoid" else ""), "tokens_per_gpu": T, "global_tokens": T * world, "hidden": d,
                   "ffn": f, "experts": E, "top_k": k, "shared_experts": NS, "gating": gating, "format": "(N,M,V)=(%d,%d,%d) + 2:4" % FMT + (" (run as plain 2:4)" if cfg.kernel_config() is not cfg
                                                               else ""),
                   "parallelism": ((f"ep{world} (experts sharded; token rows / outputs over NVLink peer memory "
                                    "inside the SSMM kernels, tags over NCCL)" if transport == "peer" else
                                    f"ep{world} (experts sharded; dispatch/combine by torch all_to_all_single)"
                                    if transport == "torch" else
                                    f"ep{world} (experts sharded; dispatch/combine by the library's NCCL "
                                    "communicator, grouped ncclSend/Recv inside samoyeds_moe_layer)") if ep
                                   else f"dp{world} (experts replicated per GPU)"),
                   "l2": "inputs larger than L2: %.0f MB of compressed expert weights streamed per step"
                         % (3 * active * f * d * BYTES_PER_ELEM / 1e6),
                   "weights": "random-init (counter-based synthetic), magnitude-pruned to (%d,%d,%d)" % FMT,
                   "launch": ("cuda graph of the K timed layer calls (no phase-event nodes inside; per-phase "
                              "times from a second replay that records them)") if use_graph else "eager launches"},
        "layer_tflops": flops_layer / (ms * 1e-3) / 1e12,
        "phases_ms": {"route_compact": ph_ms[0], "zero_out": ph_ms[1], "gate_up_ssmm": ph_ms[2],
                      "down_ssmm": ph_ms[3]},
        "down_ssmm_tflops": (flops_gu / 2) / (ph_ms[3] * 1e-3) / 1e12,
        "roofline": roof,
        "e2e": {"value": T * world / (ms_e2e * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": T * d * 2 + T * lg.shape[1] * 4, "d2h_bytes_per_step": T * d * (2 if e2e_bf16 else 4),
                "out_dtype": "bf16" if e2e_bf16 else "f32",
                "overlap": "copies of steps s+1 / s-1 on separate streams beside step s (double-buffered)"},
        "decode": dec,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(model)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def nt_pick(tokens_per_expert):
    """Token tile the library picks (moe.cu: mean + 3 sigma tokens per expert, then
    the smallest NW=1, M=2 tile of ssmm.cu's table that holds it)."""
    hi = tokens_per_expert + int(3.0 * tokens_per_expert ** 0.5 + 0.999)
    for nt in (16, 32, 64, 128, 224):
        if nt >= hi:
            return nt
    return 224


def gate_up_kernel(tokens_per_expert, f):
    """Name of the interleaved gate/up SSMM kernel the library launches (moe.cu /
    ssmm.cu: ssmm_pick_nt, ssmm_pair_cluster) -- the key into the ncu summary."""
    nt = nt_pick(tokens_per_expert)
    if tokens_per_expert >= 64 and nt in (128, 224):
        return "ssmm_pair_kernel<%d, 1, 2, 1>" % nt   # <NT, NW, MS, SPLIT>: SEL-gather launches split rings
    return "ssmm_kernel<%d, 1, 2, 1>" % nt


def ncu_traffic(model, T, kernel, shared=0):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, per
    launch, from the committed ncu --set full capture of this workload
    (profiles/r2_ncu_summary.json, written by probes/ncu_summary.py from
    probes/capture_r2.sh), keyed by the kernel name the library reports
    (smy_moe_kernel_names); (None, why) when there is no capture."""
    for rnd in ("r2", "r1"):
        p = os.path.join(ROOT, "profiles", f"{rnd}_ncu_summary.json")
        if not os.path.exists(p):
            continue
        tag = "%s_T%d%s: void %s" % (model, T, f"_sh{shared}" if shared else "", kernel)
        for key, v in json.load(open(p))["kernels"].items():
            if key.startswith(tag):
                return v["dram_read"] + v["dram_write"], f"profiles/{rnd}_ncu_summary.json [{key}]"
    return None, f"no ncu capture of {model} T={T} {kernel} in profiles/"


class stdout_to_stderr:
    """Point file descriptor 1 at stderr (native libraries print banners there)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def C_void_p_array(events):
    import ctypes as C
    arr = (C.c_void_p * len(events))(*[C.c_void_p(ev.cuda_event) for ev in events])
    return arr


def set_format(spec: str):
    """--format N,M,V: the weight format of the run (module-level FMT / byte count)."""
    global FMT, BYTES_PER_ELEM
    n, m, v = (int(t) for t in spec.split(","))
    FMT = (n, m, v)
    # canonical bytes per logical element: values (N/M)/2 x 2 B + codes (N/M)/2 x 2 bit + indices (N/M)/V x 1 B
    BYTES_PER_ELEM = (n / m) * (0.5 * 2 + 0.5 * 0.25 + 1.0 / v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="mixtral", choices=sorted(MODELS))
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the timed steps eagerly instead of a CUDA graph")
    ap.add_argument("--format", default="1,2,32", help="(N,M,V) weight format (default the paper's (1,2,32))")
    ap.add_argument("--transcode", default="auto", choices=["auto", "off"],
                    help="formats without fast kernels: re-encode as plain 2:4 (auto) or keep (off)")
    ap.add_argument("--force-ep", action="store_true", help=argparse.SUPPRESS)  # EP code path at world 1 (tests)
    ap.add_argument("--parallel", default="ep", choices=["ep", "dp"], help="N>1: expert (default) or data parallel")
    ap.add_argument("--ep-transport", default="nccl", choices=["nccl", "torch", "peer"],
                    help="EP token/output transport: the library's NCCL communicator (default), torch "
                         "all_to_all_single, or NVLink peer memory inside the kernels")
    ap.add_argument("--e2e-f32", action="store_true", help="e2e leg with the fp32 layer output (default bf16)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch / process-group / timing path only, on CPU (gloo): prints the contract line")
    ap.add_argument("--shared", type=int, default=0,
                    help="shared experts (every token, weight 1) after the routed ones, e.g. 2 for DeepSeek-MoE")
    ap.add_argument("--gate-up", default="auto", choices=["auto", "interleaved", "separate"],
                    help="gate/up weight layout (auto: the library's choice for the format)")
    ap.add_argument("--shared-gate", default="none", choices=["none", "sigmoid"],
                    help="shared experts weighted 1 (default) or by a per-token sigmoid gate (Qwen2-MoE: "
                         "--model qwen2 --shared 8 --shared-gate sigmoid = its width-20480 shared expert)")
    ap.add_argument("--decode-tokens", type=int, default=64, help="extra decode point on the same layer (0: off)")
    args = ap.parse_args()
    set_format(args.format)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    if "NCCL_DEBUG" not in os.environ and args.gpus > 1:
        # communicator setup lines (rank / nranks) on stderr; stdout keeps the JSON line
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

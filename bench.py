"""bench.py — outer-step throughput of the SparseLoCo hot path on B200.

One step = one SparseLoCo outer step on this rank's FSDP shard (§2.1):
  slc_compress (Eq. 1: pseudo-gradient, EF, chunk Top-k, 2-bit Q, pack, EF residual)
  [N > 1: NCCL all-gather of the shard payloads into the peer message, overlapped]
  slc_outer_update fused (Eq. 2: decode + aggregate R peer payloads + theta update)
Metric (BASELINE.json): outer-step params/s (whole job) and HBM GB/s (% of roofline).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl slc|reference]
Under torchrun one process per GPU; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name -> (layout, R peers, param dtype)
WORKLOADS = {
    "llama3.2-1b": ("llama3.2-1b", 8, "f32"),      # BASELINE configs[1]
    "llama3-8b": ("llama3-8b", 20, "f32"),         # BASELINE configs[2]
    "covenant-72b": ("covenant-72b", 20, "f32"),   # BASELINE configs[3] (reading A, R#22)
    "covenant-72b-b": ("covenant-72b-b", 20, "f32"),  # reading B: untied, every matrix 64x64-blocked
    "llama2-7b": ("llama2-7b", 20, "f32"),         # BASELINE configs[4] base point
    "1m": ("1m-2d", 1, "f32"),                     # BASELINE configs[0]
    "flat-1b": ("flat-1b", 8, "f32"),              # bandwidth probe (contiguous chunks)
    "tiny": ("llama-tiny", 4, "f32"),              # debugging
}

BETA = 0.95
ALPHA = 1.0
SPECIAL_PERIOD = 0  # set from --special-period


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None)
    ap.add_argument("--R", type=int, default=None)
    ap.add_argument("--dtype", default=None, choices=[None, "f32", "bf16"])
    ap.add_argument("--impl", default="slc", choices=["slc", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--shard-of", type=int, default=0,
                    help="N=1 only: run shard --shard-rank of an N-way FSDP sharding (one GPU's share of a larger job)")
    ap.add_argument("--shard-rank", type=int, default=0)
    ap.add_argument("--cold-ef", action="store_true", help="round 0: e = 0 (with bf16 params many magnitudes tie)")
    ap.add_argument("--special-period", type=int, default=0,
                    help="1/P of the 4096-element runs degenerate (zero, constant, ties, ...; slcgen)")
    ap.add_argument("--block", type=int, default=64, help="chunk side B (C = B*B; P:88 uses 64)")
    ap.add_argument("--k", type=int, default=64, help="values per full chunk (P:176: 64)")
    ap.add_argument("--median-norm", action="store_true",
                    help="median-norm weights (P:101): exact payload norms + all-reduce + weighted fused update")
    ap.add_argument("--ef-offload", nargs="?", const="pipelined", default=None, choices=["serial", "pipelined"],
                    help="row f3 (P:118-132): EF in pinned host memory, swapped in for compress and out every "
                         "step; serial = whole-shard swap-in, compress, swap-out overlapping the update; "
                         "pipelined (default) = per-piece H2D / compress / D2H pipeline")
    ap.add_argument("--index-code", action="store_true",
                    help="row f4: also time slc_index_rank (colex index code, R#28) on the step's records")
    ap.add_argument("--ef-pieces", type=int, default=16, help="pieces of the pipelined EF swap (row f3)")
    ap.add_argument("--gather", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1, row a8: p2p = records pushed into every rank's message over NVLink peer memory by "
                         "the compress kernel (slc_compress_multi + device barrier); nccl = all_gather_into_tensor")
    ap.add_argument("--agg-kernel", default="auto", choices=["auto", "batch", "pipe", "simple"],
                    help="decode / fused-update implementation (SLC_OPT_AGG_KERNEL; auto = batched where it applies)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """`nvidia-smi -lms 100` in the background while the timed region runs:
    SM clock median / max and any throttle reasons seen."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [[v.strip() for v in ln.split(",")] for ln in self.out.strip().splitlines()]
        rows = [r for r in rows if len(r) == 6]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def ncu_traffic(kernel: str, workload: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu
    --set full capture (profiles/ncu_traffic.json), if it was taken on this
    workload; else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        e = t.get(kernel)
        if e and e.get("workload", "llama3.2-1b") == workload:
            return e["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def peak_hbm():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------------------- inputs
class ShardState:
    """This rank's device buffers: theta (shared global params), theta_local and
    e of the own peer, and the own records — synthetic, from slcgen."""

    def __init__(self, plan, layout, seed, peer, dtype, warm_ef, records=None):
        import torch
        self.plan, self.layout, self.seed, self.peer, self.warm = plan, layout, seed, peer, warm_ef
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        dev = torch.device("cuda", plan.device)
        n = plan.shard_elems
        self.theta = torch.zeros(n, dtype=tdt, device=dev)
        self.theta_local = torch.zeros(n, dtype=tdt, device=dev)
        self.ef = torch.zeros(n, dtype=torch.float32, device=dev)
        self.records = records if records is not None else torch.zeros(plan.payload_bytes, dtype=torch.uint8,
                                                                        device=dev)
        self.reset()

    def fill(self, buf, what, peer):
        import numpy as np
        import slcgen
        offs = np.cumsum([0] + [int(np.prod(s)) for _, s in self.layout])
        for s in self.plan.segments:
            slcgen.fill_cuda(buf[s.shard_offset:s.shard_offset + s.n_elems], what, self.seed, peer,
                             int(offs[s.tensor]) + s.tensor_begin, warm_ef=self.warm,
                             special_period=SPECIAL_PERIOD)

    def reset(self, peer=None):
        import slcgen
        p = self.peer if peer is None else peer
        self.fill(self.theta, slcgen.WHAT_THETA, p)
        self.fill(self.theta_local, slcgen.WHAT_THETA_LOCAL, p)
        self.fill(self.ef, slcgen.WHAT_EF, p)


def make_peer_records(plan, layout, shard, seed, n_peers, first_peer, dtype):
    """Simulated peers' payload slices for this shard: each peer compresses its
    own (theta, theta_local_r, e_r) — produced with the same kernel, untimed."""
    import torch
    out = []
    for r in range(first_peer, first_peer + n_peers):
        shard.reset(peer=r)
        rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=shard.theta.device)
        plan.compress(shard.theta, shard.theta_local, shard.ef, rec, beta=BETA)
        out.append(rec)
    torch.cuda.synchronize()
    return out


# --------------------------------------------------------------------------- slc arm
def run_slc(args):
    import torch
    import torch.distributed as dist

    import slcgen
    from paper_2603_08163_b200 import slc
    from paper_2603_08163_b200 import dist as sdist

    global SPECIAL_PERIOD
    SPECIAL_PERIOD = args.special_period
    slc.Plan.default_options = {slc.OPT_AGG_KERNEL: slc.AGG_KERNELS[args.agg_kernel]}
    rank, world, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # more NCCL channels / larger P2P chunks: measured 1.3-1.5x on the a8 all-gather and the a9
        # all-to-all at these message sizes on B200 (tools/coll_bench.py, profiles/r02_collectives.txt)
        os.environ.setdefault("NCCL_MIN_NCHANNELS", "64")
        os.environ.setdefault("NCCL_P2P_NET_CHUNKSIZE", "524288")
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload or ("llama3.2-1b" if world == 1 else "llama3-8b")
    lname, R, dtype = WORKLOADS[wl]
    R = args.R or R
    dtype = args.dtype or dtype
    layout = slcgen.layouts.LAYOUTS[lname]
    if args.shard_of:
        assert world == 1, "--shard-of simulates one rank of a larger job on one GPU"
        plan = slc.Plan(layout, geom=slc.geometry(args.block, args.k), rank=args.shard_rank,
                        nranks=args.shard_of, dtype=dtype, device=local)
    else:
        plan = slc.Plan(layout, geom=slc.geometry(args.block, args.k), rank=rank, nranks=world, dtype=dtype,
                        device=local)
    gather = pmsg = None
    if world > 1:
        if args.gather == "p2p":
            pmsg = sdist.PeerMessage(plan)
        gather = sdist.PayloadGather(plan)  # also the a8 reference timing in `collectives`
    own_records = pmsg.records if pmsg is not None else (gather.alloc_records() if gather else None)
    shard = ShardState(plan, layout, seed=0, peer=0, dtype=dtype, warm_ef=not args.cold_ef, records=own_records)
    peers = make_peer_records(plan, layout, shard, seed=0, n_peers=R - 1, first_peer=1, dtype=dtype)
    shard.reset()
    recs = [shard.records[:plan.payload_bytes]] + peers
    mnorm = sdist.MedianNorm(plan, R, device=dev) if args.median_norm else None
    hdrs = ([slc.make_header(plan, bytes([r + 1]) * 16, base_round=1) for r in range(R)]
            if args.median_norm else None)

    stream = torch.cuda.current_stream()
    offload = None
    if args.ef_offload:
        from paper_2603_08163_b200.offload import EFOffload
        offload = EFOffload(plan, device=dev, n_pieces=args.ef_pieces)
        offload.host.copy_(shard.ef.cpu())
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def step(i=None):
        pipelined = offload is not None and args.ef_offload == "pipelined"
        ef = offload.swap_in(stream) if offload is not None and not pipelined else shard.ef
        if i is not None:
            ev[i][0].record(stream)
        if pipelined:  # compress_ms then includes the exposed part of the swaps
            offload.compress_pipelined(shard.theta, shard.theta_local, shard.records, beta=BETA, stream=stream)
        elif pmsg is not None:  # a8 folded into compress: records pushed to every rank's message
            pmsg.compress(shard.theta, shard.theta_local, ef, beta=BETA, stream=stream)
        else:
            plan.compress(shard.theta, shard.theta_local, ef, shard.records, beta=BETA, stream=stream)
        if i is not None:
            ev[i][1].record(stream)
        if offload is not None and not pipelined:
            offload.swap_out(stream)
        if gather is not None and pmsg is None:
            gather.start(shard.records)
        if mnorm is not None:
            w = mnorm(recs, hdrs=hdrs, stream=stream)
            plan.outer_update(shard.theta, ALPHA, records=recs, hdrs=hdrs, weights_dev=w, stream=stream)
        else:
            plan.outer_update(shard.theta, ALPHA, records=recs, stream=stream)
        if pmsg is not None:
            pmsg.wait(stream)  # every rank's shard is in every rank's message
        elif gather is not None:
            gather.wait()
        if offload is not None:
            offload.wait(stream)
        if i is not None:
            ev[i][2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = plan.get_status()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            step(i)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = plan.get_status()
    if st != slc.OK:
        raise RuntimeError(f"device status {slc.status_string(st)}")
    ms_total = t0.elapsed_time(t1)
    ms_compress = sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps
    ms_update = sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps
    t = torch.tensor([ms_total, ms_compress, ms_update], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, ms_compress, ms_update = t.tolist()
    ms_step = ms_total / args.steps

    extra = {}
    if world > 1:
        rec_for_gather = gather.alloc_records()
        rec_for_gather[:plan.payload_bytes].copy_(shard.records[:plan.payload_bytes])
        extra = time_collectives(plan, gather, rec_for_gather, R, stream, dev, pmsg=pmsg)
        extra["a8_in_step"] = ("p2p: slc_compress_multi pushes each record into every rank's peer message over NVLink "
                               "(symmetric memory) + a device barrier; no collective" if pmsg is not None else
                               "nccl: all_gather_into_tensor overlapped with the fused update")

    info = plan.info
    P_total = info.total_elems
    rb = info.record_bytes
    pb = 4 if dtype == "f32" else 2
    n_local = sum(s.n_elems for s in plan.segments)
    # algorithmic bytes: compress reads theta, theta_local, e, writes e + own records;
    # fused update reads R records + theta, writes theta
    comp_bytes = n_local * (2 * pb + 8) + info.n_chunks * rb
    upd_bytes = n_local * 2 * pb + R * info.n_chunks * rb
    peak, peak_src = peak_hbm()
    comp_gbs = comp_bytes / (ms_compress * 1e-3) / 1e9
    step_gbs_rank = (comp_bytes + upd_bytes) / (ms_step * 1e-3) / 1e9

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, plan, shard, recs, stream)
        if world > 1:  # whole job: the slowest rank
            tm = torch.tensor([e2e["ms_per_step"]], dtype=torch.float64, device=dev)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            e2e["ms_per_step"] = tm.item()
        e2e = {"value": (n_local if args.shard_of else P_total) / (e2e["ms_per_step"] * 1e-3), **e2e}

    out = {
        "metric": "outer-step params/s",
        "value": (n_local if args.shard_of else P_total) / (ms_step * 1e-3),
        "unit": "params/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32" if dtype == "f32" else "bf16-params/f32-ef",
        "data": "synthetic (slcgen: seeded Llama-shaped param sets; random-init values)",
        "config": {"workload": f"{wl} ({P_total} params), R={R} peers, C={args.block ** 2} k={args.k} 2-bit, "
                               f"beta={BETA} alpha={ALPHA}",
                   "params": P_total, "peers": R, "parallelism": f"fsdp-shard{world}",
                   "agg_kernel": args.agg_kernel, **({"gather": args.gather} if world > 1 else {}),
                   "l2": "inputs > L2 (126 MB): no flush needed"},
        "hbm_gbs": step_gbs_rank * world,
        "hbm_frac_of_peak": step_gbs_rank / peak,
        "roofline": {"bound": "hbm", "kernel": "slc_compress", "achieved": comp_gbs, "peak": peak,
                     "unit": "GB/s", "frac": comp_gbs / peak,
                     "frac_of_8tbs": comp_gbs / 8000.0,
                     "traffic": (ncu_traffic("compress", wl) if R == WORKLOADS[wl][1] and args.block == 64
                                 and args.k == 64 and not args.shard_of else None),
                     "traffic_source": ("not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum "
                                        "per launch from the committed ncu --set full capture "
                                        "(profiles/ncu_traffic.json) of the same kernel on this workload"),
                     "algorithmic_bytes_per_launch": comp_bytes, "peak_source": peak_src},
        "step_roofline": {"achieved_gbs_per_gpu": step_gbs_rank, "frac_of_measured_peak": step_gbs_rank / peak,
                          "frac_of_8tbs": step_gbs_rank / 8000.0,
                          "bytes_per_param": (comp_bytes + upd_bytes) / max(1, n_local),
                          "note": "whole step (compress + fused update) algorithmic bytes / step time, per GPU; "
                                  "north_star's roofline is 8 TB/s per GPU"},
        "kernels": {"compress_ms": ms_compress, "fused_update_ms": ms_update,
                    "compress_bytes_per_launch": comp_bytes, "update_bytes_per_launch": upd_bytes},
        # per step: compress = the warp-specialised kernel + the deferred-chunk
        # fallback kernel (C 1024 / 4096; one kernel at C 16384), per piece when
        # pipelined; then payload norms + weights (median-norm) + the fused update
        "gpu_launches": ((2 if plan.geom.block * plan.geom.block in (1024, 4096) else 1)
                         * (len(offload.pieces) if offload is not None and args.ef_offload == "pipelined" else 1)
                         + (3 if args.median_norm else 1)) * args.steps,
        "clocks": clk.summary(),
    }
    if args.index_code:
        out["index_code"] = time_index_rank(plan, shard, stream, R, recs)
    if offload is not None:
        out["config"]["ef_offload"] = {"mode": args.ef_offload, "pieces": len(offload.pieces),
                                       **time_offload(offload, stream, reps=3)}
    if args.special_period:
        out["config"]["special_period"] = args.special_period
    if args.cold_ef:
        out["config"]["ef"] = "cold (round 0, e = 0)"
    if args.median_norm:
        out["config"]["median_norm"] = ("P:101: exact payload norms (slc_payload_sqnorm) + int64 all-reduce + "
                                        "lower-median weights on device + weighted fused update; in the timed step")
    if args.shard_of:
        out["config"]["shard"] = (f"rank {args.shard_rank} of {args.shard_of} ({n_local} params on this GPU); "
                                  "value = this shard's params / step time")
    if e2e is not None:
        out["e2e"] = e2e
    if extra:
        out["collectives"] = extra
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(layout, R, dtype, args.cpu_seconds)
    if world > 1:
        dist.destroy_process_group()
    return out if rank == 0 else None


def time_index_rank(plan, shard, stream, R, recs, reps=5):
    """Row f4 (not in the timed step): the colex rank alone, the entropy-coded
    record encode / decode (GPU unrank) of one payload, and the update fed by
    entropy-coded payloads (R decodes + the fused update) against the update
    on fixed-width records."""
    import torch
    dev = shard.records.device
    ranks = torch.empty(plan.n_chunks * 16, dtype=torch.int32, device=dev)
    ec = torch.empty(plan.n_chunks * plan.ec_record_bytes, dtype=torch.uint8, device=dev)
    tmp = [torch.empty(plan.payload_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    plan.index_rank(shard.records, ranks, stream=stream)  # prepares the binomial table once
    plan.index_encode(shard.records, ec, stream=stream)
    torch.cuda.synchronize()

    def timed(fn, n=reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    rank_ms = timed(lambda: plan.index_rank(shard.records, ranks, stream=stream))
    enc_ms = timed(lambda: plan.index_encode(shard.records, ec, stream=stream))
    dec_ms = timed(lambda: plan.index_decode(ec, tmp[0], stream=stream))
    th = shard.theta.clone()
    upd_ms = timed(lambda: plan.outer_update(th, ALPHA, records=recs, stream=stream), 3)
    if plan.get_status() != 0:
        raise RuntimeError("index code: device status")
    del th
    return {"rank_ms": rank_ms, "encode_ms": enc_ms, "decode_ms": dec_ms, "chunks": plan.n_chunks,
            "record_bytes": plan.record_bytes, "ec_record_bytes": plan.ec_record_bytes,
            "payload_bytes": plan.payload_bytes, "ec_payload_bytes": plan.n_chunks * plan.ec_record_bytes,
            "update_fixed_width_ms": upd_ms, "update_from_ec_ms": R * dec_ms + upd_ms, "R": R,
            "note": "R#28: 15 rank limbs + codes + scales per chunk (80 B vs 116 B); decode = greedy colex "
                    "unranking, a 32-way warp search per position; update_from_ec = R decodes + the fused update "
                    "(the record bytes the update reads drop 31 %, the unranking costs far more: P:91-93's "
                    "'significant overhead')"}


def time_offload(offload, stream, reps=3):
    """Row f3: the two EF swaps timed alone on the copy stream (host-link bound, 4 B/param each way)."""
    import torch
    cs = offload.copy_stream
    res = {}
    for name, fn in (("swap_in", lambda: offload.swap_in(stream)), ("swap_out", lambda: offload.swap_out(stream))):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cs)
            fn()
            b.record(cs)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        res[name + "_ms"] = ms
        res[name + "_gbs"] = offload.bytes_per_swap / (ms * 1e-3) / 1e9
    res["bytes_each_way"] = offload.bytes_per_swap
    res["note"] = ("P:118-132: EF lives in pinned host memory between steps; serial step = swap-in + compress + "
                   "max(swap-out, fused update); pipelined step ~ max(swap-in, swap-out) + update tail; the swaps "
                   "are host-link bound; swap_* timed alone, whole shard")
    return res


def time_collectives(plan, gather, records, R, stream, dev, reps=5, pmsg=None):
    """a8 all-gather of the shard payloads alone, and the a9 simulated-peer
    exchange (peer r's full message on rank r % n; each rank receives its slice
    of every message) — both max over ranks, reported beside the step."""
    import torch
    import torch.distributed as dist
    from paper_2603_08163_b200 import dist as sdist
    world, rank = dist.get_world_size(), dist.get_rank()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    gather.start(records)
    gather.wait()
    torch.cuda.synchronize()
    dist.barrier()
    a.record(stream)
    for _ in range(reps):
        gather.start(records)
        gather.wait()
    b.record(stream)
    torch.cuda.synchronize()
    ag_ms = a.elapsed_time(b) / reps
    ex = sdist.PeerExchange(gather, R)
    owned = [gather.message for _ in range(rank, R, world)]  # every peer message: same bytes, same size
    for i, m in enumerate(owned):
        ex.stage(i, m)  # where the download would have written them

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    ex_ms = timed(ex.exchange)
    p2p_ms = timed(lambda: ex.run_p2p(owned))
    del ex
    exp = sdist.PeerExchangeP2P(plan, gather.sizes, gather.slot, R)
    for i, m in enumerate(owned):
        exp.stage(i, m)
    pull_ms = timed(lambda: exp.exchange(stream))
    del exp
    agp_ms = 0.0
    if pmsg is not None:  # a8 data movement alone over NVLink: pull every other rank's slot
        local = torch.empty(world * pmsg.slot, dtype=torch.uint8, device=dev)
        base = [int(pmsg.handle.buffer_ptrs[g]) for g in range(world)]
        pairs = [(base[g] + g * pmsg.slot, local.data_ptr() + g * pmsg.slot, pmsg.sizes[g])
                 for g in range(world) if g != rank]

        def pull():
            pmsg.handle.barrier(channel=0)
            plan.peer_copy(pairs, stream=stream)

        agp_ms = timed(pull)
        del local
    t = torch.tensor([ag_ms, ex_ms, p2p_ms, pull_ms, agp_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ag_ms, ex_ms, p2p_ms, pull_ms, agp_ms = t.tolist()
    moved = R * plan.payload_bytes * (world - 1) / world  # bytes per rank that cross NVLink
    msg = sum(gather.sizes)
    return {"allgather_ms": ag_ms, "allgather_message_bytes": msg,
            "allgather_busbw_gbs": msg * (world - 1) / world / (ag_ms * 1e-3) / 1e9,
            **({"allgather_pull_ms": agp_ms,
                "allgather_pull_busbw_gbs": msg * (world - 1) / world / (agp_ms * 1e-3) / 1e9} if agp_ms else {}),
            "exchange_ms": ex_ms, "exchange_bytes_per_rank": R * plan.payload_bytes,
            "exchange_gbs_per_rank": moved / (ex_ms * 1e-3) / 1e9,
            "exchange_p2p_ms": p2p_ms, "exchange_pull_ms": pull_ms,
            "exchange_pull_gbs_per_rank": moved / (pull_ms * 1e-3) / 1e9,
            "exchange_method": "staged all_to_all_single (one NCCL call); p2p = grouped send/recv per (peer, dst) "
                               "slice; pull = every rank pulls its slices from the owners' symmetric-memory "
                               "messages over NVLink with one slc_peer_copy kernel between two device barriers",
            "note": "all-gather overlapped with the fused update inside the step; exchange (stand-in for the "
                    "R2 download) reported separately, not in ms_per_step"}


def run_e2e(args, plan, shard, recs, stream):
    """Same step through the public API with host buffers: every step copies
    the step's inputs (theta_local, the R-1 peer payloads) from pinned host
    memory and reads back the own payload (to upload) — copies inside the timer."""
    import torch
    n = plan.shard_elems
    tl_host = torch.empty(n, dtype=shard.theta_local.dtype, pin_memory=True)
    tl_host.copy_(shard.theta_local)
    peer_host = [r.cpu().pin_memory() for r in recs[1:]]
    own_host = torch.empty(plan.payload_bytes, dtype=torch.uint8, pin_memory=True)
    h2d = tl_host.numel() * tl_host.element_size() + sum(p.numel() for p in peer_host)
    d2h = own_host.numel()
    steps = max(2, min(args.steps, 5))

    def step():
        shard.theta_local.copy_(tl_host, non_blocking=True)
        for d, h in zip(recs[1:], peer_host):
            d.copy_(h, non_blocking=True)
        plan.compress(shard.theta, shard.theta_local, shard.ef, shard.records, beta=BETA, stream=stream)
        plan.outer_update(shard.theta, ALPHA, records=recs, stream=stream)
        own_host.copy_(recs[0], non_blocking=True)

    step()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    return {"unit": "params/s", "ms_per_step": ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps}


# --------------------------------------------------------------------------- oracle (CPU) arm
_CPU_SAMPLE = None  # the oracle sample, inherited by forked workers


def _oracle_worker(args):
    """One host core: cycle over its share of the sample for `seconds`."""
    wid, nworkers, seconds = args
    import oracle
    g = oracle.geom()
    mine = _CPU_SAMPLE[wid::nworkers] or _CPU_SAMPLE[:1]
    work, steps, params = 0.0, 0, 0
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end:
        for a, l, e, peers, n in mine:
            t0 = time.perf_counter()
            st, rec, en = oracle.compress_chunk(a, l, e, BETA, g)
            delta = oracle.aggregate_chunk([rec] + peers, n, g=g)
            oracle.outer_update(a, delta, ALPHA)
            work += time.perf_counter() - t0
            steps += 1
            params += n
            if time.perf_counter() >= t_end:
                break
    return work, steps, params


def _cpu_info():
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    aff = sorted(os.sched_getaffinity(0))
    return model, os.cpu_count(), aff


def cpu_baseline(layout, R, dtype, seconds, pool=256):
    """The oracle as it stands (oracle/slco.c, single-threaded C, untuned) on a
    bounded sample of the workload, on every host core of this process's
    affinity mask: per chunk-step = compress the own chunk + aggregate R
    records (own + R-1 peers) + outer update, over a deterministic pool of
    `pool` chunks drawn across all tensors (peer records precomputed, untimed);
    chunks are independent, so T forked workers each cycle over a
    disjoint share for `seconds` of wall time.  params/s = all params done /
    wall time.  A single-core run of seconds/4 is reported beside it."""
    global _CPU_SAMPLE
    import multiprocessing as mp

    import numpy as np

    import oracle
    import slcgen
    g = oracle.geom()
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in layout])
    allc = [(ti, c) for ti, (_, shape) in enumerate(layout) for c in range(oracle.tensor_chunks(shape, g))]
    rng = np.random.default_rng(0)
    pick = sorted(rng.choice(len(allc), size=min(pool, len(allc)), replace=False).tolist())
    sample = []
    for i in pick:
        ti, c = allc[i]
        off = oracle.chunk_offsets(layout[ti][1], c, g)
        G = offs[ti] + off
        a = slcgen.generate_at(0, 0, 0, G, dtype=dtype)
        l = slcgen.generate_at(1, 0, 0, G, dtype=dtype)
        e = slcgen.generate_at(2, 0, 0, G, warm_ef=True)
        peers = []
        for r in range(1, R):
            st, rec, _ = oracle.compress_chunk(a, slcgen.generate_at(1, 0, r, G, dtype=dtype),
                                               slcgen.generate_at(2, 0, r, G, warm_ef=True), BETA, g)
            peers.append(rec)
        sample.append((a, l, e, peers, len(off)))
    _CPU_SAMPLE = sample
    model, ncpu, aff = _cpu_info()
    T = max(1, len(aff))
    w1, s1, p1 = _oracle_worker((0, 1, max(1.0, seconds / 4)))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(T) as pl:
        res = pl.map(_oracle_worker, [(w, T, seconds) for w in range(T)])
    wall = time.perf_counter() - t0
    steps = sum(r[1] for r in res)
    params = sum(r[2] for r in res)
    return {"value": params / wall, "unit": "params/s", "cores": T, "kind": "oracle",
            "sample": f"{steps} chunk-steps over a pool of {len(sample)} chunks drawn from all {len(layout)} tensors "
                      f"({params} params), R={R}; per chunk: compress own + aggregate R records + update; the "
                      f"single-threaded C oracle on {T} forked workers (disjoint chunk shares), {wall:.1f} s wall",
            "single_thread_value": p1 / w1, "single_thread_seconds": w1,
            "cpu_model": model, "cpu_count": ncpu, "affinity": aff, "wall_seconds": wall}


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on the host cores."""
    rank, world, local = dist_env()
    if rank != 0:
        return None
    wl = args.workload or ("llama3.2-1b" if world == 1 else "llama3-8b")
    lname, R, dtype = WORKLOADS[wl]
    R = args.R or R
    dtype = args.dtype or dtype
    import slcgen
    layout = slcgen.layouts.LAYOUTS[lname]
    per_step = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(layout, R, dtype, per_step, pool=128)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    P = slcgen.layouts.total_params(layout)
    return {"impl": "reference", "metric": "outer-step params/s", "value": v, "unit": "params/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": P / v * 1e3,
            "extrapolated": True,
            "extrapolation": f"each step runs the oracle on a bounded sample ({cb['sample']}); ms_per_step = "
                             f"{P} params / the measured params/s (a full step would take {P / v:.0f} s)",
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic (slcgen)",
            "config": {"workload": f"{wl} ({P} params), R={R} peers, C=4096 k=64 2-bit", "params": P, "peers": R},
            "cpu_baseline": {**cb, "value": v},
            "e2e": {"value": v, "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    out = run_reference(args) if args.impl == "reference" else run_slc(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

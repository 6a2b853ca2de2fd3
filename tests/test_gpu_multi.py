"""Multi-GPU path over NCCL (rows a8, a9, e, f1): one process per GPU, each
compressing, gathering, exchanging and updating its own FSDP shard (P:88,
P:112-116), checked against the single-GPU path and the oracle.

* a8: the all-gathered peer message equals the 1-GPU plan's records of the
  same inputs byte for byte (and the oracle's, for the ragged layout);
* a9: every rank's received slice of every simulated peer's message equals
  that peer's records for the rank's shard;
* e:  every rank's theta slice after the fused outer step equals the oracle
  (whole shard for the ragged layout, sampled chunks for llama-tiny);
* f1: MedianNorm's weights over NCCL (int64 limb all-reduce) equal the
  1-GPU weights of the full messages bitwise, and the weighted update equals
  the oracle with those weights.
Skipped when fewer GPUs than the world size are visible."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA devices", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layout_name, dtype, R, sample, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    res = {"rank": rank}
    try:
        import oracle
        from helpers import bits, make_device_inputs, oracle_compress_shard, oracle_update_shard, seg_view
        from paper_2603_08163_b200 import slc
        from paper_2603_08163_b200.dist import MedianNorm, PayloadGather, PeerExchange
        from slcgen import layouts
        layout = layouts.LAYOUTS[layout_name]
        plan = slc.Plan(layout, rank=rank, nranks=world, dtype=dtype, device=rank)
        full = slc.Plan(layout, rank=0, nranks=1, dtype=dtype, device=rank)
        gather = PayloadGather(plan, device=dev)
        seed = 7
        theta = None
        own, messages, full_recs = [], [], []
        for r in range(R):
            theta, tl, ef = make_device_inputs(plan, layout, seed, r, dtype, special_period=16, warm_ef=True,
                                               theta=theta)
            rec = gather.alloc_records()
            plan.compress(theta, tl, ef, rec)
            own.append(rec[:plan.payload_bytes].clone())
            gather.start(rec)
            gather.wait()
            messages.append(gather.message.clone())            # padded: rank g's part at g * slot
            # the same peer on one GPU
            th1, tl1, ef1 = make_device_inputs(full, layout, seed, r, dtype, special_period=16, warm_ef=True)
            rec1 = torch.zeros(full.payload_bytes, dtype=torch.uint8, device=dev)
            full.compress(th1, tl1, ef1, rec1)
            full_recs.append(rec1)
        torch.cuda.synchronize()
        plan.check()
        # a8: gathered message == 1-GPU records
        res["a8"] = all(torch.equal(torch.cat([m[g * gather.slot:g * gather.slot + gather.sizes[g]]
                                               for g in range(world)]), f)
                        for m, f in zip(messages, full_recs))
        if sample is None:  # and == the oracle's records of the whole layout
            ok = True
            for r in range(R):
                ref, _, _ = oracle_compress_shard(full, layout, seed, r, dtype, special_period=16, warm_ef=True)
                ok &= np.array_equal(full_recs[r].cpu().numpy().view(np.uint32), ref)
            res["a8_oracle"] = ok
        # a8 over NVLink peer memory: compress pushes every record into every rank's message
        try:
            from paper_2603_08163_b200.dist import PeerMessage
            pm = PeerMessage(plan)
            ok = True
            for r in range(R):
                th_, tl_, ef_ = make_device_inputs(plan, layout, seed, r, dtype, special_period=16, warm_ef=True,
                                                   theta=theta)
                pm.compress(th_, tl_, ef_)
                pm.wait()
                torch.cuda.synchronize()
                ok &= torch.equal(pm.contiguous_message(), full_recs[r])
                dist.barrier()
            res["a8_p2p"] = ok
        except Exception:
            import traceback
            res["a8_p2p_error"] = traceback.format_exc()[-1500:]
        # a9: peer r's padded message lives on rank r % world
        ex = PeerExchange(gather, R)
        slices = ex.run([messages[r] for r in range(rank, R, world)])
        torch.cuda.synchronize()
        res["a9"] = all(torch.equal(s, o) for s, o in zip(slices, own))
        try:  # a9 pulled over NVLink peer memory
            from paper_2603_08163_b200.dist import PeerExchangeP2P
            exp = PeerExchangeP2P(plan, gather.sizes, gather.slot, R)
            sl2 = exp.run([messages[r] for r in range(rank, R, world)])
            torch.cuda.synchronize()
            res["a9_p2p"] = all(torch.equal(s, o) for s, o in zip(sl2, own))
        except Exception:
            import traceback
            res["a9_p2p_error"] = traceback.format_exc()[-1500:]
        # e: fused outer step on the shard vs the oracle
        alpha = 0.65
        th0 = theta.clone()
        plan.outer_update(theta, alpha, records=slices)
        plan.check()
        ref_recs = [s.cpu().numpy().view(np.uint32) for s in slices]
        thetas_host = [seg_view(th0, s).cpu() for s in plan.segments]
        if dtype == "bf16":
            thetas_host = [t.view(torch.int16).numpy().view(np.uint16) for t in thetas_host]
        else:
            thetas_host = [t.numpy() for t in thetas_host]
        res["e"] = _compare_update(plan, theta, thetas_host, ref_recs, alpha, None, sample, dtype)
        # f1: median-norm weights over NCCL vs the 1-GPU weights of the full messages
        mn = MedianNorm(plan, R, device=dev)
        w = mn(slices).clone()
        sq = torch.zeros((R, 4), dtype=torch.int64, device=dev)
        full.payload_sqnorm(full_recs, sq)
        w1 = torch.zeros(R, dtype=torch.float32, device=dev)
        full.median_norm_weights(sq, w1)
        torch.cuda.synchronize()
        res["f1_weights"] = torch.equal(w.view(torch.int32), w1.view(torch.int32))
        th2 = th0.clone()
        plan.outer_update(th2, alpha, records=slices, weights_dev=w)
        plan.check()
        res["f1_update"] = _compare_update(plan, th2, thetas_host, ref_recs, alpha, w.cpu().numpy(), sample, dtype)
    except Exception as exc:  # reported through the queue
        import traceback
        res["error"] = traceback.format_exc()[-3000:]
    finally:
        q.put(res)
        dist.destroy_process_group()


def _compare_update(plan, theta_dev, thetas_host, ref_recs, alpha, weights, sample, dtype):
    import oracle
    from helpers import bits, oracle_update_shard, seg_view
    from slcgen import layouts  # noqa: F401
    g = oracle.geom()
    RW = oracle.record_words(g)
    if sample is None:
        ref = oracle_update_shard(plan, thetas_host, ref_recs, alpha, weights=weights)
        for s, t in zip(plan.segments, ref):
            got = seg_view(theta_dev, s).cpu()
            if dtype == "bf16":
                got = got.view(torch.int16)
            if not np.array_equal(bits(got.numpy()), bits(t)):
                return False
        return True
    # sampled chunks: oracle on single chunks of the shard
    rng = np.random.default_rng(plan.info.rank)
    off = 0
    ok = True
    for s, th in zip(plan.segments, thetas_host):
        shape = (s.rows, s.cols) if s.blocked else (s.n_elems,)
        nc = oracle.tensor_chunks(shape, g)
        for c in sorted(rng.choice(nc, min(nc, sample), replace=False).tolist()):
            per = [rr[(off + c) * RW:(off + c + 1) * RW] for rr in ref_recs]
            new = oracle.aggregate_update_tensor(shape, th, [np.tile(p, 1) for p in per], alpha,
                                                 weights=weights, c0=c, c1=c + 1, g=g)
            idx = oracle.chunk_offsets(shape, c, g)
            got = seg_view(theta_dev, s).cpu()
            if dtype == "bf16":
                got = got.view(torch.int16)
            got = bits(got.numpy())[idx]
            ok &= np.array_equal(got, bits(new)[idx])
        off += nc
    return ok


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("layout_name,dtype,R,sample", [("ragged", "f32", 5, None), ("ragged", "bf16", 3, None),
                                                        ("llama-tiny", "f32", 6, 3)])
def test_nccl_gather_exchange_update(world, layout_name, dtype, R, sample):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout_name, dtype, R, sample, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    errs = [r[k] for r in res for k in r if k.endswith("error")]
    assert not errs, errs[0]
    for r in res:
        for k, v in r.items():
            if k != "rank":
                assert v is True or v == True, (r["rank"], k, r)  # noqa: E712

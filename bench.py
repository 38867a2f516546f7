#!/usr/bin/env python
"""Benchmark of the B200 activation compressor (BASELINE.json metric).

metric : compress+decompress GB/s per B200 at eb=1e-3 (% of HBM peak); compression ratio
step   : one round trip (compress, then decompress with the zero filter) of the whole
         saved-activation set of the workload, inputs resident in HBM.
basis  : algorithmic bytes B = 8n + 2C per round trip: read 4n fp32 and
         write C ACZ1 bytes (compress), read C and write 4n (decompress).
value  : total B over all ranks / max-over-ranks device time of the K timed steps.

Default workload is configs[1]: AlexNet saved-activation set, batch 256 (407 MB), on one
B200. Multi-GPU (torchrun): each rank compresses its own batch-256 set (weak scaling, no
collective on the data path; the only collectives are the barrier and the max-reduce of
the timings).

--impl reference times the reference's own CPU implementation (oracle/_ref, compiled from
the reference sources) on the host cores: each step is a bounded sample of the same
workload, batch-sharded over all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EB = 1e-3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="alexnet",
                    choices=["alexnet", "config1", "vgg16", "resnet18", "resnet50"])
    ap.add_argument("--batch", type=int, default=0, help="per-rank batch (0: workload default)")
    ap.add_argument("--eb", type=float, default=EB)
    ap.add_argument("--data", default="iid", choices=["iid", "smooth", "model"],
                    help="synthetic activations: iid (default), smooth (box-filtered), or "
                         "model (a random-initialised AlexNet/VGG-16 forward pass)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    return ap.parse_args()


DEFAULT_BATCH = {"alexnet": 256, "config1": 64, "vgg16": 256, "resnet18": 1024, "resnet50": 512}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------------- clocks ----
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------- our arm ----
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2011_09017_b200 as acz
    from paper_2011_09017_b200 import _native, workloads as W
    import ctypes as C

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    batch = args.batch or DEFAULT_BATCH[args.workload]
    # weak scaling: every rank holds a full per-rank batch (rank-seeded)
    tensors = [x for _, x in W.make_set(args.workload, batch * max(world, 1), device=dev,
                                        shard=(rank, max(world, 1)), data=args.data)]
    names = [nm for nm, _, _ in W.activation_set(args.workload)]
    n_total = sum(x.numel() for x in tensors)
    outs = [torch.empty_like(x) for x in tensors]
    ctx = acz.default_context(local_rank)
    lib = _native.load()
    stream = torch.cuda.current_stream()
    params = acz.CodecParams(args.eb)

    def step():
        # the whole activation set through the batched entry points (one call each way)
        blobs = acz.compress_many(tensors, params, stream=stream, ctx=ctx)
        acz.decompress_many(blobs, zero_filter=True, outs=outs, stream=stream)
        return sum(c.compressed_bytes for c in blobs), blobs

    # nvidia-smi needs ~0.1-0.3 s to start sampling: start it before the warm-up so the
    # samples cover the (short) timed region; warm-up steps run the same load
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = lib.acz_gpu_launch_count(ctx.handle)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    cbytes = 0
    for _ in range(args.steps):
        cb, blobs = step()
        cbytes = cb
        del blobs
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    launches = int(lib.acz_gpu_launch_count(ctx.handle) - l0)
    clk = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(8 * n_total + 2 * cbytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms_max = t.item()
    B_all = tot.item()  # bytes per step over all ranks
    value = B_all * args.steps / (ms_max * 1e-3) / 1e9

    # ---- compress and decompress timed separately (4n/T_c and 4n/T_d; an
    # extra pass after the timed region, events on the launching stream) ----
    split = None
    if world == 1:
        tc = td = 0.0
        reps = max(3, min(args.steps, 10))
        for _ in range(reps):
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a2 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            bl = acz.compress_many(tensors, params, stream=stream, ctx=ctx)
            a1.record(stream)
            acz.decompress_many(bl, zero_filter=True, outs=outs, stream=stream)
            a2.record(stream)
            torch.cuda.synchronize()
            tc += a0.elapsed_time(a1)
            td += a1.elapsed_time(a2)
            del bl
        tc /= reps
        td /= reps
        split = {"compress_ms": tc, "decompress_ms": td,
                 "compress_gbps_4n": 4 * n_total / (tc * 1e-3) / 1e9,
                 "decompress_gbps_4n": 4 * n_total / (td * 1e-3) / 1e9,
                 "note": "compress_many and decompress_many timed separately (events); "
                         "4n / T over the fp32 activation bytes (SURVEY 8(d))"}

    # ---- per-kernel times (separate passes with event timing around every launch) ----
    kms = (C.c_double * 7)()
    kn = (C.c_uint64 * 7)()
    kclass = ["stats", "quant", "histogram", "codebook", "encode", "decode", "scan"]
    # per-tensor, per-class times (tensors one at a time, so every launch is timed alone):
    # the dominant single kernel of the step for the roofline
    per_tensor = []
    for nm, x, o in zip(names, tensors, outs):
        lib.acz_gpu_profile_enable(ctx.handle, 1)
        c = acz.compress(x, params, stream=stream, ctx=ctx)
        acz.decompress(c, zero_filter=True, out=o, stream=stream)
        torch.cuda.synchronize()
        lib.acz_gpu_profile_read(ctx.handle, kms, kn)
        per_tensor.append((nm, x.numel(), c.compressed_bytes,
                           {kclass[i]: kms[i] for i in range(7) if kn[i]}))
    lib.acz_gpu_profile_enable(ctx.handle, 0)
    # per-class totals from the isolated passes: in the batched step the tensors' streams
    # overlap and priority queueing stretches the event brackets of the short kernels
    kern = {}
    for nm, n_t, C_t, d in per_tensor:
        for cls, ms in d.items():
            e = kern.setdefault(cls, {"ms_per_step": 0.0, "launches_per_step": 0.0})
            e["ms_per_step"] += ms
            e["launches_per_step"] += 1.0

    # per-tensor detail (one extra pass, not timed)
    detail = []
    ratios_in, ratios_out = 0, 0
    for nm, x in zip(names, tensors):
        c = acz.compress(x, params, stream=stream, ctx=ctx)
        detail.append({"tensor": nm, "shape": list(x.shape), "ratio": round(acz.compression_ratio(c), 4),
                       "book": c.codebook_size, "outliers": c.outlier_count,
                       "max_len": c.max_code_length})
        ratios_in += c.uncompressed_bytes
        ratios_out += c.compressed_bytes

    host = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        host = host_set(args, tensors)  # the CPU baseline runs on these exact bytes
    # memory the codec holds (what compression is for): blobs of one step (ACZ1 payload +
    # decode sidecars + tables) and this context's workspace after the batched step
    blobs = acz.compress_many(tensors, params, stream=stream, ctx=ctx)
    torch.cuda.synchronize()
    mem = ctx.memory_info()
    memory = {"activation_bytes": 4 * n_total,
              "acz1_bytes": sum(c.compressed_bytes for c in blobs),
              "blob_device_bytes": sum(c.device_bytes for c in blobs),
              "workspace_bytes": mem["workspace_bytes"],
              "workspace_breakdown": mem["workspace_breakdown"]}
    del blobs
    ctx.trim()
    memory["workspace_bytes_after_trim"] = ctx.memory_info()["workspace_bytes"]
    res = dict(host=host, value=value, ms_per_step=ms_max / args.steps, n=n_total, cbytes=cbytes,
               memory=memory, split=split,
               B_step=8 * n_total + 2 * cbytes, launches=launches, clocks=clk, kernels=kern,
               detail=detail, ratio=ratios_in / ratios_out, batch=batch, per_tensor=per_tensor)

    # ---- e2e through the public host-buffer API (page-locked host memory in and out) ----
    # every rank runs it at once (each GPU through its own host link), timed per rank on the
    # host around synchronised steps; the job's value is all ranks' bytes / the slowest rank
    if not args.no_e2e:
        hin = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in tensors]
        for h, x in zip(hin, tensors):
            h.copy_(x)
        hout = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in tensors]
        bbufs = [torch.empty(5 * x.numel() + (1 << 20), dtype=torch.uint8, pin_memory=True)
                 for x in tensors]
        sbufs = [torch.empty(x.numel() // 8 + (1 << 20), dtype=torch.uint8, pin_memory=True)
                 for x in tensors]

        def e2e_step():
            res_b = acz.compress_host_many(hin, params, blob_bufs=bbufs, side_bufs=sbufs, ctx=ctx,
                                           stream=stream)
            acz.decompress_host_many(res_b, zero_filter=True, outs=hout, ctx=ctx, stream=stream)
            cb = sum(b.size for b, _ in res_b)
            sb = sum(sd.size for _, sd in res_b)
            h2d = sum(h.numel() * 4 for h in hin) + cb + sb
            d2h = cb + sb + sum(h.numel() * 4 for h in hout)
            return h2d, d2h, cb

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            h2d, d2h, cb = e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        agg = torch.tensor([dt, float(8 * n_total + 2 * cb), float(h2d), float(d2h)],
                           dtype=torch.float64, device=dev)
        if world > 1:
            mx = agg[:1].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(agg, op=dist.ReduceOp.SUM)
            agg[0] = mx[0]
        dt, b_all, h2d, d2h = agg[0].item(), agg[1].item(), int(agg[2].item()), int(agg[3].item())
        res["e2e"] = {"value": b_all * args.e2e_steps / dt / 1e9, "unit": "GB/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ranks": world,
                      "path": "compress_host_many + decompress_host_many (C-ABI "
                              "acz_gpu_compress_host_batch / acz_gpu_decompress_host_batch; "
                              "page-locked host buffers, copies inside the timed region)"}
        # bit-exactness spot check of the e2e path against the device path
        res["e2e"]["matches_device_path"] = bool(all(torch.equal(h.to(dev), o)
                                                     for h, o in zip(hout, outs)))
    return res


# ------------------------------------------------------------------ CPU reference ----
TRAFFIC_JSON = os.path.join("profiles", "r02", "v7", "traffic.json")
ONE_THREAD_SAMPLES = 16  # 1-thread leg: the first 16 samples of every tensor (~2-3 s)


def _cuda() -> bool:
    import torch
    return torch.cuda.is_available()


def host_set(args, tensors=None):
    """The GPU arm's exact input bytes on the host: workloads.make_set (torch Philox on
    cuda:0, seed 20201118 + tensor index) copied down, or the given device tensors."""
    import torch
    from paper_2011_09017_b200 import workloads as W
    if tensors is None:
        batch = args.batch or DEFAULT_BATCH[args.workload]
        dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
        tensors = [x for _, x in W.make_set(args.workload, batch, device=dev, data=args.data)]
    return [x.cpu().numpy() for x in tensors]


def cpu_reference_sample(args, host, threads=None):
    """The reference CPU codec (oracle/_ref, compiled from the reference sources) on the
    whole per-GPU batch of every tensor (the GPU arm's bytes), compress + decompress with the
    zero filter, batch-sharded into `threads` shards on `threads` host threads (the
    reference's functions are pure; one codebook per shard).
    Returns (GB/s on basis B = 8n + 2C, detail)."""
    from oracle.oracle import Reference
    R = Reference()
    threads = threads or os.cpu_count() or 1
    tot_B, tot_s, n_tot = 0, 0.0, 0
    for x in host:
        cb, sec = R.roundtrip_sharded(x, args.eb, shards=threads, threads=threads)
        tot_B += 8 * x.size + 2 * cb
        tot_s += sec
        n_tot += x.size
    return tot_B / tot_s / 1e9, {"threads": threads, "samples_per_tensor": host[0].shape[0],
                                 "elements": n_tot, "seconds": tot_s}


def cpu_reference_one_thread(args, host, samples=ONE_THREAD_SAMPLES):
    """The reference's own usage, one thread: acz::compress + acz::decompress of each
    (whole, unsharded) tensor of a bounded sample (the first `samples` samples of every
    tensor, same bytes as the GPU arm). Returns (GB/s on basis B, detail)."""
    from oracle.oracle import Reference
    R = Reference()
    tot_B, tot_s, n_tot = 0, 0.0, 0
    for x in host:
        xs = x[:samples]
        cb, sec = R.roundtrip_sharded(xs, args.eb, shards=1, threads=1)
        tot_B += 8 * xs.size + 2 * cb
        tot_s += sec
        n_tot += xs.size
    return tot_B / tot_s / 1e9, {"threads": 1, "samples_per_tensor": samples,
                                 "elements": n_tot, "seconds": tot_s}


def cpu_baseline_lines(args, host):
    v, info = cpu_reference_sample(args, host)
    v1, info1 = cpu_reference_one_thread(args, host)
    return {"value": v, "unit": "GB/s", "cores": info["threads"], "kind": "reference",
            "sample": f"all {info['samples_per_tensor']} samples of every {args.workload} tensor "
                      f"(the GPU arm's input bytes), {info['threads']} batch shards on "
                      f"{info['threads']} threads ({info['seconds']:.2f} s)",
            "one_thread": {"value": v1, "unit": "GB/s", "cores": 1,
                           "sample": f"first {info1['samples_per_tensor']} samples of every "
                                     f"tensor, whole-tensor compress+decompress "
                                     f"({info1['seconds']:.2f} s)"}}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle.oracle import reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    batch = args.batch or DEFAULT_BATCH[args.workload]
    host = host_set(args)
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        v, info = cpu_reference_sample(args, host)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    v1, info1 = cpu_reference_one_thread(args, host)
    line = {
        "metric": "compress+decompress GB/s per B200 at eb=1e-3 (% of HBM peak); compression ratio",
        "impl": "reference", "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": f"synthetic ({args.data})",
        "config": {"workload": f"{args.workload} saved-activation set, batch {batch} per GPU, "
                               f"fp32, eb={args.eb}, zero filter on decompress",
                   "input": ("the GPU arm's bytes (workloads.make_set, Philox on cuda:0)"
                             if _cuda() else "workloads.make_set on the CPU generator "
                                              "(no GPU: not the GPU arm's bytes)"),
                   "sample": f"{info['samples_per_tensor']} samples per tensor per step"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": info["threads"],
                         "kind": "reference",
                         "sample": f"all {info['samples_per_tensor']} samples of every "
                                   f"{args.workload} tensor ({info['elements']} elements), "
                                   f"{info['threads']} batch shards on {info['threads']} threads",
                         "one_thread": {"value": v1, "unit": "GB/s", "cores": 1,
                                        "sample": f"first {info1['samples_per_tensor']} samples "
                                                  f"of every tensor, whole-tensor compress + "
                                                  f"decompress"}},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------- main ----
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # ACZ_BENCH_ONE_GPU=1 (testing the multi-rank path on a one-GPU box): every rank on cuda:0,
    # gloo for the barrier / max-reduction; the numbers are not a scaling measurement
    one_gpu = os.environ.get("ACZ_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        peak, kind = load_peaks()
        kern = res["kernels"]
        # roofline of the dominant single kernel launch of the step: algorithmic bytes of
        # that launch (quantiser reads 4n, histogram reads the symbols, encode
        # writes C, decode reads C and writes 4n) / its event-timed duration
        alg_of = {"quant": lambda n, C: 4 * n, "histogram": lambda n, C: 2 * n,
                  "encode": lambda n, C: 2 * n + C, "decode": lambda n, C: C + 4 * n,
                  "codebook": lambda n, C: 0, "stats": lambda n, C: 4 * n}
        best = max(((nm, n_t, C_t, cls, ms) for nm, n_t, C_t, d in res["per_tensor"]
                    for cls, ms in d.items()), key=lambda r: r[4])
        dnm, dn, dC, dom, dms = best
        dalg = alg_of.get(dom, lambda n, C: 0)(dn, dC)
        achieved = dalg / (dms * 1e-3) / 1e9 if dms > 0 else 0.0
        traffic = None  # measured DRAM bytes of that launch, from the committed ncu capture
        if args.workload == "alexnet" and dnm == "conv1_in" and dom == "quant" and args.eb == EB:
            try:
                with open(os.path.join(ROOT, TRAFFIC_JSON)) as f:
                    traffic = json.load(f)["dram_bytes_per_launch"]
            except Exception:  # noqa: BLE001
                traffic = None
        line = {
            "metric": "compress+decompress GB/s per B200 at eb=1e-3 (% of HBM peak); compression ratio",
            "value": res["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": f"synthetic ({args.data})",
            "config": {"workload": f"{args.workload} saved-activation set, batch {res['batch']} per "
                                   f"GPU, fp32, eb={args.eb}, zero filter on decompress",
                       "parallelism": f"dp{world} (batch-sharded, no data-path collective)",
                       "l2": "inputs (%.0f MB/GPU) exceed the 126 MB L2" % (4 * res["n"] / 1e6),
                       "basis": "B = 8n + 2C algorithmic bytes per round trip"},
            "pct_hbm": res["value"] / world / peak,
            "compression_ratio": res["ratio"],
            "roofline": {"bound": "hbm", "kernel": f"{dom} ({dnm})", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_kind": kind,
                         "algorithmic_bytes_per_launch": dalg, "launch_ms": dms,
                         "traffic_source": f"{TRAFFIC_JSON} (ncu --set full)",
                         "roundtrip_frac": res["value"] / world / peak},
            "kernels": kern,
            "kernels_basis": "per class, summed over the tensors each compressed + decompressed "
                             "alone with CUDA events around every launch",
            "gpu_launches": res["launches"],
            "memory": res["memory"],
            "compress_decompress_split": res.get("split"),
            "clocks": res["clocks"],
            "detail": res["detail"],
        }
        if "e2e" in res:
            line["e2e"] = res["e2e"]
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline_lines(args, res["host"])
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"unavailable": str(e)}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

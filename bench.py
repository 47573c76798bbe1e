#!/usr/bin/env python
"""COBS query / build benchmark on B200 (see DESIGN.md §6 for the contract).

Default workload: BASELINE.json config 5 -- the 100,000-document compact
index (~100 GB, resident in HBM) queried with 100,000 random 1,000-bp
queries at K = 0.8.  One step = one batch of the whole query set through
kernels 1-3.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                    [--config c5|c1] [--queries Q]

Arms:
  gpu (default)  value: inputs resident in HBM; e2e: the reference-facing
                 C-ABI call with host (pinned) patterns, H2D + D2H inside the
                 timed region.  Adds roofline, cpu_baseline, build.
  reference      the reference's own CPU implementation (oracle/_ref: the
                 unmodified /root/reference sources) on the host cores, on a
                 bounded sample of the same workload.
Multi-GPU: weak scaling -- every rank holds its own replica of the index and
queries its own batch (no data-path collective).
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

import numpy as np  # noqa: E402

METRIC = "query q-grams/sec and row-gather HBM GB/s (fraction of peak); docs/sec index build"
UNIT = "q-grams/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--config", default="c5", choices=["c5", "c1"])
    ap.add_argument("--queries", type=int, default=0, help="override the batch size")
    ap.add_argument("--cpu-sample", type=int, default=0, help="queries in the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-build", action="store_true")
    ap.add_argument("--c5-median", type=float, default=0.0)
    ap.add_argument("--c5-docs", type=int, default=0)
    ap.add_argument("--c5-block-size", type=int, default=0)
    ap.add_argument("--shard", default="replicas", choices=["replicas", "blocks"],
                    help="replicas: every rank holds the whole index and answers its own batch "
                         "(weak scaling); blocks: every rank holds a block range of the C5 index "
                         "and answers the whole batch, hit lists merged on rank 0 (strong scaling)")
    ap.add_argument("--engine", default="cuda", choices=["cuda", "oracle"],
                    help=argparse.SUPPRESS)  # oracle: CPU test of the launcher/exchange only
    return ap.parse_args()


CPU_SAMPLE = 1024  # queries (ids 0..CPU_SAMPLE-1) of the CPU legs: cpu_baseline and --impl reference


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def world_info(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch with "
                         f"--nproc-per-node {args.gpus}, or without a launcher)")
    return rank, world, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_traffic(workload: str):
    """Per-launch DRAM traffic of the gather kernel from the committed ncu
    capture (profiles/), scaled per algorithmic byte, or None."""
    path = os.path.join(ROOT, "profiles", "gather_ncu_traffic.json")
    try:
        d = json.load(open(path))
        if d.get("workload") != workload:
            return None
        return d
    except Exception:
        return None


# ---------------------------------------------------------------- helpers

def c5_config(args):
    from workloads import synth
    cfg = synth.CONFIGS["c5"]
    if args.c5_median:
        cfg = synth.replace(cfg, c5_median=args.c5_median)
    if args.c5_docs:
        cfg = synth.replace(cfg, n_docs=args.c5_docs)
    if args.c5_block_size:
        cfg = synth.replace(cfg, block_size=args.c5_block_size)
    if args.queries:
        cfg = synth.replace(cfg, n_queries=args.queries)
    return cfg


def host_available_bytes() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 0


def c5_payload_bytes(cfg) -> int:
    """File payload of the C5 index (what an in-RAM copy needs)."""
    from oracle import oracle as O
    orc = O.OracleIndex.c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
    return sum(w * ((dc + 7) // 8) for dc, w, _ in orc.blocks())


def open_ref_c5(cfg, cores):
    """The reference view of the C5 index: an in-RAM copy (the reference's
    resident layout) when the host has room for it with 15 % headroom, else
    the procedural IndexView that regenerates rows per call (slower; labelled)."""
    from oracle import oracle as O
    need = c5_payload_bytes(cfg)
    materialise = host_available_bytes() > need * 1.15
    ref = O.RefIndex.c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p,
                        materialise=materialise, threads=cores)
    how = ("an in-RAM copy of the same index" if materialise else
           "the procedural view (rows regenerated per call; host RAM too small for an in-RAM copy)")
    return ref, how


def workload_name(cfg):
    if cfg.name == "c5":
        return (f"c5: compact {cfg.n_docs}-document index (log-normal term counts, median "
                f"{cfg.c5_median:.3g}, sigma {cfg.c5_sigma}), {cfg.n_queries} random {cfg.qlen}-bp "
                f"queries, K={cfg.K}")
    return (f"{cfg.name}: {'classic' if cfg.kind == 0 else 'compact'} {cfg.n_docs} docs, "
            f"{cfg.n_queries} x {cfg.qlen}-bp queries, K={cfg.K}")


def build_c1_index(cfg, device):
    """Config-1 index built on the device from the seeded corpus."""
    import paper_1905_09624_b200 as cb
    from workloads import synth
    buf, off = synth.docs(cfg)
    names = synth.doc_names(cfg)
    docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
    img = cb.build_classic(docs, cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p), device=device)
    return cb.open_image(img, device)


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's own CPU query path (oracle/_ref = unmodified
    /root/reference sources), threaded over all host cores.  This process
    loads nothing outside oracle/: the inputs come from the oracle library's
    copy of the seeded generator (workloads.synth.bind), never from the
    product package."""
    from oracle import oracle as O
    from workloads import synth
    O.ensure_built()
    synth.bind(O.ORACLE_SO)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    if args.config == "c5":
        cfg = c5_config(args)
        t0 = time.perf_counter()
        ref, how = open_ref_c5(cfg, cores)
        setup_s = time.perf_counter() - t0
        per_step = args.cpu_sample or CPU_SAMPLE
        K = cfg.K
    else:
        cfg = synth.CONFIGS["c1"]
        import tempfile
        buf, off = synth.docs(cfg)
        names = synth.doc_names(cfg)
        docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
        t0 = time.perf_counter()
        tmp = tempfile.mkdtemp()
        O.ref_build_write(docs, os.path.join(tmp, "c1.cobs"), q=cfg.q, k=cfg.k, p=cfg.p)
        ref = O.RefIndex.open(os.path.join(tmp, "c1.cobs"))
        setup_s = time.perf_counter() - t0
        per_step = args.cpu_sample or cfg.n_queries
        K = cfg.K
        how = "the reference's open_resident of its own build"
    # every step answers the same bounded sample: query ids 0..per_step-1, the
    # ids the GPU arm's cpu_baseline times
    ids = np.arange(per_step, dtype=np.uint64) % np.uint64(cfg.n_queries)
    qb, qo = synth.queries(cfg, ids)
    times, grams = [], []
    for step in range(args.warmup + args.steps):
        t = time.perf_counter()
        ell, sk, st, nh, _ = ref.query_batch(qb, qo, K, threads=cores)
        dt = time.perf_counter() - t
        if step >= args.warmup:
            times.append(dt)
            grams.append(int(ell.sum()))
    value = sum(grams) / sum(times)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u64",
        "data": "synthetic (seeded)", "impl": "reference",
        "config": {"workload": workload_name(cfg), "step": f"{per_step}-query bounded sample (ids 0..{per_step - 1})",
                   "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"query ids 0..{per_step - 1} every step x {args.steps} steps over {how}, "
                                   f"index load {setup_s:.1f}s excluded"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- gpu arm

def cpu_baseline_c5(cfg, sample):
    from oracle import oracle as O
    from workloads import synth
    cores = os.cpu_count() or 1
    ref, how = open_ref_c5(cfg, cores)
    qb, qo = synth.queries(cfg, np.arange(sample, dtype=np.uint64))
    t = time.perf_counter()
    ell, sk, st, nh, _ = ref.query_batch(qb, qo, cfg.K, threads=cores)
    dt = time.perf_counter() - t
    ref.close()
    return {"value": float(ell.sum()) / dt, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{sample} of the batch's queries (ids 0..{sample - 1}) through the "
                      f"reference query() over {how}, {cores} threads, {dt:.1f}s"}


def run_gpu(args):
    import torch
    import paper_1905_09624_b200 as cb
    from workloads import synth

    rank, world, local = world_info(args)
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or "WORLD_SIZE" in os.environ:  # (a 1-rank torchrun still runs the NCCL exchange)
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (NVLS etc.) in the log
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.shard == "blocks":
        return run_gpu_blocks(args, rank, world, local, dist)

    if args.config == "c5":
        cfg = c5_config(args)
        t0 = time.perf_counter()
        view = cb.synth_c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma,
                           cfg.p, device=local)
    else:
        cfg = synth.CONFIGS["c1"]
        if args.queries:
            cfg = synth.replace(cfg, n_queries=args.queries)
        t0 = time.perf_counter()
        view = build_c1_index(cfg, local)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.Stream(device=local)
    view.set_stream(stream.cuda_stream)

    from paper_1905_09624_b200.dist import reduce_max, reduce_sum, weak_query_ids
    ids = weak_query_ids(cfg.n_queries, rank) if cfg.name == "c5" else np.arange(cfg.n_queries, dtype=np.uint64)
    qb, qo = synth.queries(cfg, ids)
    n = len(qo) - 1
    h_pat = torch.from_numpy(qb).pin_memory()
    h_off = torch.from_numpy(qo.view(np.int64)).pin_memory()
    d_pat = h_pat.to(f"cuda:{local}")
    d_off = h_off.to(f"cuda:{local}")
    torch.cuda.synchronize()

    def step_device():
        return cb.query_batch_raw(view, d_pat.data_ptr(), (d_off.data_ptr(), n), cfg.K,
                                  device_input=True, keep_device=True)

    def step_e2e():
        return cb.query_batch_raw(view, h_pat.numpy(), h_off.numpy().view(np.uint64), cfg.K)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            outs = [fn() for _ in range(steps)]
            e1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = reduce_max(e0.elapsed_time(e1) / steps, f"cuda:{local}")  # max over ranks
        return ms, outs

    def step_pruned():
        return cb.query_batch_raw(view, h_pat.numpy(), h_off.numpy().view(np.uint64), cfg.K, prune=True)

    clocks = ClockSampler(local)
    clocks.start()
    ms_dev, outs = timed(step_device, args.steps, args.warmup)
    ms_e2e, outs_e2e = timed(step_e2e, args.steps, 1)
    ms_pruned, outs_pruned = timed(step_pruned, args.steps, 1)
    clk = clocks.stop()

    grams = int(outs[-1].ell.astype(np.uint64).sum())
    total_grams = int(reduce_sum(grams, f"cuda:{local}"))  # q-grams of all ranks
    value = total_grams / (ms_dev / 1e3)
    e2e_value = total_grams / (ms_e2e / 1e3)
    last = outs_e2e[-1]
    h2d = int(qb.nbytes + qo.nbytes)
    d2h = int(n * (4 + 4 + 8 + 4) + last.docs.nbytes + last.scores.nbytes)

    # roofline of the dominant kernel (gather): algorithmic bytes
    # k * sum(l) * sum_b row_bytes_b per launch / its event-timed duration
    gather_ms = statistics.mean(o.ms_gather for o in outs)
    algo_bytes = outs[-1].row_bytes
    achieved = algo_bytes / (gather_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    tr = ncu_traffic(cfg.name)
    traffic = None
    if tr and tr.get("algo_bytes"):
        traffic = tr["dram_bytes"] / tr["algo_bytes"] * algo_bytes
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "kernel": "gather_kernel", "algo_bytes_per_launch": algo_bytes,
                "gather_ms": gather_ms,
                "share_of_step": gather_ms / ms_dev,
                "termize_ms": statistics.mean(o.ms_termize for o in outs),
                "order_ms": statistics.mean(o.ms_order for o in outs)}

    # same-box ceilings (after the timed region): the gather's access shape,
    # random 128-byte lines, and a streaming read, on this GPU in this process
    try:
        free, _ = torch.cuda.mem_get_info(local)
        st_gbs, rnd_gbs = cb.calibrate(local, min(16 << 30, free // 2))
        roofline["same_box"] = {"stream_read_gbs": st_gbs, "random128_gbs": rnd_gbs,
                                "frac_of_stream_read": achieved / st_gbs,
                                "frac_of_random128": achieved / rnd_gbs,
                                "what": "tools-free calibration (cobs_gpu_calibrate): random 128-byte "
                                        "lines, 16 in flight per warp, over a 16 GiB buffer"}
    except Exception as e:  # report, do not die
        roofline["same_box"] = {"error": repr(e)}

    lens = np.diff(qo.astype(np.int64))
    windows = int(np.maximum(lens - cfg.q + 1, 0).sum())
    termize_ms = statistics.mean(o.ms_termize for o in outs)
    kmer = {"kernel": "termize_hash_kernel", "ms": termize_ms, "windows": windows,
            "windows_per_s": windows / (termize_ms / 1e3),
            "hashes_per_s": cfg.k * grams / (termize_ms / 1e3),
            "bound": "integer ALU (XXH64: 19 64-bit multiplies per q=31 window)"}

    index_bytes = view.device_bytes()
    cpu_base = None
    build = None
    if rank == 0 and world == 1:
        view.close()  # the timed part is over; free HBM for the build legs
        if not args.no_build:
            build = {"c1": bench_build(cb, synth, local)}
            for name in ("c2", "c3", "c4"):
                try:
                    build[name] = bench_build_cfg(cb, synth, name, local)
                except Exception as e:
                    build[name] = {"error": repr(e)}
        if not args.no_cpu_baseline:
            try:
                if cfg.name == "c5":
                    cpu_base = cpu_baseline_c5(cfg, args.cpu_sample or CPU_SAMPLE)
                else:
                    cpu_base = cpu_baseline_c1(cfg)
            except Exception as e:  # report, do not die
                cpu_base = {"value": None, "error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_dev, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8/u64", "data": "synthetic (seeded)",
            "config": {"workload": workload_name(cfg), "queries_per_gpu": n,
                       "index_bytes_hbm": index_bytes,
                       "l2": "inputs larger than L2 (index ~100 GB, hashes ~0.8 GB)"
                             if cfg.name == "c5" else "index L2-resident (35 MB)",
                       "parallelism": f"replicas x{world} (independent query batches)",
                       "setup_s": setup_s},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e},
            "gpu_launches": int(sum(o.launches for o in outs)),
            # the same batch with threshold pruning (COBS_Q_PRUNE): a (query,
            # slice) stops reading rows once no document there can reach tau;
            # identical hit lists (checked here and in the tests), fewer bytes.
            # Not used for `value`: the headline keeps the reference's full work.
            "pruned": {"e2e_value": total_grams / (ms_pruned / 1e3), "unit": UNIT,
                       "ms_per_step": ms_pruned,
                       "gather_ms": statistics.mean(o.ms_gather for o in outs_pruned),
                       "hits_identical": bool(np.array_equal(outs_pruned[-1].docs, outs_e2e[-1].docs)
                                              and np.array_equal(outs_pruned[-1].hit_n, outs_e2e[-1].hit_n))},
            "roofline": roofline,
            # kernel 1 (q-gram extraction + canonical + XXH64 + dedup):
            # sustained window and hash throughput, event-timed per launch
            "kmer_kernel": kmer,
            "cpu_baseline": cpu_base,
            "build": build,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def cpu_baseline_c1(cfg):
    import tempfile
    from oracle import oracle as O
    from workloads import synth
    cores = os.cpu_count() or 1
    buf, off = synth.docs(cfg)
    names = synth.doc_names(cfg)
    docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
    tmp = tempfile.mkdtemp()
    O.ref_build_write(docs, os.path.join(tmp, "c1.cobs"), q=cfg.q, k=cfg.k, p=cfg.p)
    ref = O.RefIndex.open(os.path.join(tmp, "c1.cobs"))
    qb, qo = synth.queries(cfg)
    t = time.perf_counter()
    ell, *_ = ref.query_batch(qb, qo, cfg.K, threads=cores)
    dt = time.perf_counter() - t
    return {"value": float(ell.sum()) / dt, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"all {cfg.n_queries} queries, {cores} threads, {dt:.2f}s"}


BUILD_CPU_SAMPLE = {"c1": 1000, "c2": 64, "c3": 32, "c4": 256}  # documents the CPU reference builds


def cpu_reference_build(cfg, synth, n_docs: int) -> dict:
    """The reference's own build (oracle/_ref: extract_terms on every host
    core, then build_classic / build_compact + write_index) over the first
    n_docs documents of the config's corpus: a bounded sample, since its
    build API holds every TermSet in RAM."""
    import tempfile
    from oracle import oracle as O
    ids = np.arange(min(n_docs, cfg.n_docs), dtype=np.uint64)
    lengths = synth.doc_lengths(cfg)
    buf, off = synth.docs(cfg, ids, lengths=lengths)
    names = synth.doc_names(cfg, ids.tolist())
    docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(len(ids))]
    path = os.path.join(tempfile.mkdtemp(), "ref.cobs")
    t = time.perf_counter()
    O.ref_build_write(docs, path, q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical,
                      block_size=cfg.block_size, kind=cfg.kind)
    dt = time.perf_counter() - t
    os.remove(path)
    return {"docs_per_s": len(ids) / dt, "cores": os.cpu_count(), "seconds": dt,
            "sample": f"documents 0..{len(ids) - 1} of the corpus ({int(lengths[:len(ids)].sum())} bytes)",
            "what": "reference extract_terms (all cores) + build_" + ("classic" if cfg.kind == 0 else "compact")
                    + " + write_index"}


def bench_build_cfg(cb, synth, name: str, device: int) -> dict:
    """docs/s of index construction on a config's full corpus, generated in
    HBM: one warm-up build (reported as `cold`: the first build of a process
    also pays the first touch of its fresh key buffers), then the median of
    5 builds (on power-capped boxes about one fill pass in four runs 20-50 %
    long, profiles/r2/session5/ab_fillnoise.log).  `docs_per_s_kernels` counts the count + fill passes (sequences
    in HBM -> finished, queryable matrix), `docs_per_s_call` the whole call."""
    import torch
    cfg = synth.CONFIGS[name]
    lengths = synth.doc_lengths(cfg)
    dev = torch.empty(int(lengths.sum()), dtype=torch.uint8, device=f"cuda:{device}")
    cb.synth_docs_device(cfg.seed, cfg.alpha, lengths, dev.data_ptr(), device)
    seg_off = np.zeros(cfg.n_docs + 1, np.uint64)
    np.cumsum(lengths, out=seg_off[1:])
    params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical, block_size=cfg.block_size)
    names = synth.doc_names(cfg)
    torch.cuda.synchronize()
    runs = []
    index_bytes = 0
    for rep in range(6):
        view, _ = cb.build_device(dev.data_ptr(), seg_off, np.arange(cfg.n_docs + 1), names, params, cfg.kind,
                                  device=device, seqs_on_device=True)
        runs.append(cb.last_build_timing_ex())
        index_bytes = view.device_bytes()
        view.close()
    del dev
    torch.cuda.empty_cache()
    cold, warm = runs[0], runs[1:]
    med = lambda key: statistics.median(r[key] for r in warm)  # noqa: E731
    # ms_count = the whole count leg (its kernels + the cudaMalloc / cudaFree
    # of its workspace); the kernels alone are ms_count_kernels
    c, f, tot = med("ms_count_kernels"), med("ms_fill"), med("ms_total")
    windows = int(np.maximum(lengths.astype(np.int64) - cfg.q + 1, 0).sum())
    out = {"config": f"{name}: {'classic' if cfg.kind == 0 else 'compact B=%d' % cfg.block_size}, "
                     f"{cfg.n_docs} docs, q={cfg.q}, k={cfg.k}, p={cfg.p}, canonical={cfg.canonical}",
           "corpus_bytes": int(lengths.sum()), "windows": windows, "index_bytes_hbm": index_bytes,
           "docs_per_s_kernels": cfg.n_docs / ((c + f) / 1e3), "docs_per_s_call": cfg.n_docs / (tot / 1e3),
           "ms_count": c, "ms_fill": f, "ms_total_call": tot,
           "ms_count_leg": med("ms_count"), "ms_count_alloc": med("ms_count_alloc"), "ms_count_free": med("ms_count_free"),
           "runs_ms": [[r["ms_count_kernels"], r["ms_fill"], r["ms_total"]] for r in warm],
           "runs_count_alloc_free_ms": [[r["ms_count_alloc"], r["ms_count_free"]] for r in warm],
           "cold": {"ms_count": cold["ms_count_kernels"], "ms_count_leg": cold["ms_count"], "ms_fill": cold["ms_fill"],
                    "ms_total_call": cold["ms_total"]},
           # the build is integer-issue bound, not HBM bound: its HBM traffic
           # (corpus read + keys + matrix) is a small fraction of peak
           "throughput": {"count_windows_per_s": windows / (c / 1e3),
                          "fill_hashes_per_s": cfg.k * windows / (f / 1e3),
                          "algo_bytes": int(lengths.sum()) + index_bytes,
                          "algo_gbs": (int(lengths.sum()) + index_bytes) / ((c + f) / 1e3) / 1e9}}
    # Rooflines of the two passes against the measured HBM copy peak.  Neither
    # is HBM-bound: the count's design traffic (corpus rolled twice, 8-byte
    # keys written to super-buckets, re-sorted into buckets and read by the
    # dedup: 34 B per window) runs at a fraction of peak -- its kernels are
    # issue/latency bound (the histogram's and scatter's rolling, the
    # scatter's per-key 8-byte stores, the dedup sets' probe loop); the fill
    # (corpus once + the matrix written and copied) is issue-bound on the
    # IMAD pipe (XXH64's 64-bit multiplies).  ncu figures: committed captures.
    peak, _ = measured_peak()
    count_bytes = 34 * windows
    fill_bytes = int(lengths.sum()) + 3 * index_bytes
    out["roofline"] = {
        "count": {"bound": "issue/latency (rolling, per-key scattered stores, the dedup probe loop), not HBM",
                  "design_bytes": count_bytes, "achieved_gbs": count_bytes / (c / 1e3) / 1e9,
                  "peak_gbs": peak, "frac": count_bytes / (c / 1e3) / 1e9 / peak,
                  "ncu": "profiles/r2/session5/launch_build_c3_s5g.csv (C3 launch list, serialised: hist 151, "
                         "super scatter 222, final 339, dedup 289 ms; scatter / final / dedup = 0.45 / 0.52 / 0.31 "
                         "of the HBM peak on their own design bytes); per-kernel ncu details: "
                         "profiles/r2/session5/ncu/, dedup_fast_u1_details.csv"},
        "fill": {"bound": "issue (IMAD pipe: XXH64's 19 64-bit multiplies per window), not HBM",
                 "design_bytes": fill_bytes, "achieved_gbs": fill_bytes / (f / 1e3) / 1e9,
                 "peak_gbs": peak, "frac": fill_bytes / (f / 1e3) / 1e9 / peak,
                 "issue_active_frac": 0.71,
                 "ncu": "profiles/r2/fill_c3_mix.md (slab_fill_kernel, one C3 wave: 71 % issue slots busy, "
                        "288 instructions per window; round 1: 74.5 %, profiles/r1/build_fill_wave_c3_details.csv)"}}
    try:
        out["cpu_reference"] = cpu_reference_build(cfg, synth, BUILD_CPU_SAMPLE[name])
    except Exception as e:
        out["cpu_reference"] = {"error": repr(e)}
    return out


def bench_build(cb, synth, device):
    """docs/s of index construction on the config-1 corpus (1,000 x 100 kb):
    kernel time (sequences in HBM -> finished matrix) and end to end (host
    sequences -> file image in host memory); warm-up + median of 3."""
    cfg = synth.CONFIGS["c1"]
    buf, off = synth.docs(cfg)
    names = synth.doc_names(cfg)
    docs = [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
    params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p)
    cb.build_classic(docs, params, device=device)  # warm-up
    runs = []
    for _ in range(3):
        t = time.perf_counter()
        cb.build_classic(docs, params, device=device)
        runs.append((cb.last_build_timing_ex(), time.perf_counter() - t))
    runs.sort(key=lambda r: r[0]["ms_count_kernels"] + r[0]["ms_fill"])
    t, wall = runs[1]  # the median of 3
    c, f, tot = t["ms_count_kernels"], t["ms_fill"], t["ms_total"]
    out = {"config": "c1: classic, 1,000 docs x 100,000 bp, k=1, p=0.3",
           "docs_per_s_kernels": cfg.n_docs / ((c + f) / 1e3),
           # host sequences -> H2D -> kernels -> index file image in host memory
           "docs_per_s_e2e": cfg.n_docs / (tot / 1e3),
           "ms_h2d": t["ms_h2d"], "ms_count": c, "ms_fill": f, "ms_d2h_image": t["ms_d2h"],
           "ms_total_device_call": tot, "ms_wall": 1e3 * wall}
    try:
        out["cpu_reference"] = cpu_reference_build(cfg, synth, BUILD_CPU_SAMPLE["c1"])
    except Exception as e:
        out["cpu_reference"] = {"error": repr(e)}
    return out


def run_gpu_blocks(args, rank, world, local, dist):
    """--shard blocks: the C5 index split by blocks over the ranks (an index
    larger than one GPU, e.g. the literal-median 185 GB C5 over 2+ GPUs).
    Every rank answers the whole batch on its blocks; one step = local
    kernels 1-3, the hit lists to the host, the tensor all_gather of the hit
    lists (NCCL) and the rank-0 merge by (score desc, name asc).  Strong
    scaling: the batch and the index are fixed, N GPUs share them."""
    import torch
    import paper_1905_09624_b200 as cb
    from workloads import synth
    from paper_1905_09624_b200.dist import (all_gather_arrays, flat_hits, gather_block_hits, name_ranks, reduce_max,
                                            shard_range)
    if args.config != "c5":
        raise SystemExit("--shard blocks serves the compact C5 index")
    cfg = c5_config(args)
    nb = (cfg.n_docs + cfg.block_size - 1) // cfg.block_size
    b_lo, b_hi = shard_range(nb, rank, world)
    t0 = time.perf_counter()
    view = cb.synth_c5_blocks(cfg.seed, b_lo, b_hi, cfg.n_docs, cfg.block_size, cfg.c5_median,
                              cfg.c5_sigma, cfg.p, device=local)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.Stream(device=local)
    view.set_stream(stream.cuda_stream)
    off = view.column_offset()
    # rank 0 ranks every column's name (the merge's tie-break); each shard
    # knows its own columns' names only -- C5 names are "doc" + the zero-padded
    # draw index, so the draw indices are gathered once (setup, untimed)
    ids = np.array([int(nm[3:]) for nm in view.doc_names()], np.int64)
    parts = all_gather_arrays([ids], f"cuda:{local}")
    name_rank = None
    if rank == 0:
        width = max(6, len(str(cfg.n_docs - 1)))
        name_rank = name_ranks([b"doc" + str(int(c)).zfill(width).encode()
                                for c in np.concatenate([p[0] for p in parts])])
    qb, qo = synth.queries(cfg)
    n = len(qo) - 1
    dev = f"cuda:{local}"

    def step():
        r = cb.query_batch_raw(view, qb, qo, cfg.K)
        hn, cols, sc = flat_hits(r)
        merged = gather_block_hits(hn, cols + off, sc, name_rank, 0, dev)
        return r, merged

    for _ in range(args.warmup):
        step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t = time.perf_counter()
    outs = [step() for _ in range(args.steps)]
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / args.steps * 1e3
    if dist:
        dist.barrier()
    ms = reduce_max(wall, dev)
    grams = int(outs[-1][0].ell.astype(np.uint64).sum())  # every shard sees the whole batch
    if rank == 0:
        line = {
            "metric": METRIC, "value": grams / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8/u64", "data": "synthetic (seeded)",
            "config": {"workload": workload_name(cfg), "queries": n,
                       "parallelism": f"block shards x{world} (blocks {b_lo}..{b_hi - 1} on rank 0 of {nb})",
                       "index_bytes_hbm_rank0": view.device_bytes(), "setup_s": setup_s,
                       "timing": "host wall clock per step (kernels + hit D2H + NCCL all_gather + merge), "
                                 "max over ranks"},
            "hits_total": int(outs[-1][1][0].sum()),
        }
        print(json.dumps(line), flush=True)
    view.close()
    if dist:
        dist.destroy_process_group()
    return 0


def run_oracle_engine(args):
    """Test-only (--engine oracle): the launcher, the world-size check, the
    max-over-ranks timing and the block-shard exchange of the GPU arm, with
    the CPU oracle answering each rank's share (gloo; no GPU).  Never a bench
    number."""
    import torch.distributed as tdist
    from oracle import oracle as O
    from workloads import synth
    from paper_1905_09624_b200.dist import gather_block_hits, name_ranks, reduce_max, shard_range
    rank, world, _ = world_info(args)
    dist = None
    if world > 1:
        tdist.init_process_group("gloo")
        dist = tdist
    cfg = c5_config(args)
    idx = O.OracleIndex.c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
    names = idx.names()
    blocks = idx.blocks()
    b_lo, b_hi = shard_range(len(blocks), rank, world)
    col_lo, col_hi = blocks[b_lo][2], blocks[b_hi - 1][2] + blocks[b_hi - 1][0]
    qb, qo = synth.queries(cfg)
    n = len(qo) - 1
    t = time.perf_counter()
    hn, cols, sc, grams, full = [], [], [], 0, []
    for i in range(n):
        ell, _, h, _ = idx.query(qb[int(qo[i]):int(qo[i + 1])].tobytes(), cfg.K)
        grams += ell
        full.append(h)
        mine = [(d, s_) for d, s_ in h if col_lo <= d < col_hi] if args.shard == "blocks" else h
        hn.append(len(mine))
        cols += [d for d, _ in mine]
        sc += [s_ for _, s_ in mine]
    merged = gather_block_hits(np.asarray(hn, np.int64), np.asarray(cols, np.int64), np.asarray(sc, np.int64),
                               name_ranks(names), 0) if args.shard == "blocks" else None
    ms = reduce_max((time.perf_counter() - t) * 1e3)
    if rank == 0:
        ok = None
        if merged is not None:
            want = [(d, s_) for h in full for d, s_ in h]
            ok = list(zip(merged[1].tolist(), merged[2].tolist())) == want
        print(json.dumps({"metric": METRIC, "value": grams / (ms / 1e3), "unit": UNIT, "n_gpus": world,
                          "steps": 1, "warmup": 0, "ms_per_step": ms, "engine": "oracle (test only)",
                          "shard": args.shard, "hits_identical": ok}), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.engine == "oracle":
        return run_oracle_engine(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""Benchmark: sampled tokens/s of the ezLDA three-branch hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config pubmed] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step is one full iteration of the hot path (word-prep, doc pass + MPT skip test,
three-branch sampler + W/n_k rebuild, and the W all-reduce when N > 1) over the
whole synthetic corpus (every token counts, skipped or not).  The corpus
is generated on the GPU (seeded planted-LDA recipe), partitioned into
contiguous token-balanced document ranges, one range per rank; the
total corpus is fixed as N grows ("strong" scaling).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2007_08725_b200.synth import CONFIGS, CORPUS_SEED, SAMPLER_SEED  # noqa: E402

METRIC = "sampled tokens/s"
UNIT = "tokens/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.out = out
        return False

    def summary(self):
        if self.proc is None or not getattr(self, "out", ""):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_sample(cfg, target_tokens: int, seed: int = CORPUS_SEED):
    """A bounded sample of the same workload for the CPU oracle: the planted-LDA recipe of
    the config with the config's vocabulary and doc-length law, n_docs chosen so the sample
    holds ~target_tokens (numpy generator)."""
    from paper_2007_08725_b200.synth import planted_corpus_np

    n_docs = max(1, int(round(target_tokens / cfg.mean_len)))
    w, d = planted_corpus_np(n_docs, cfg.V, cfg.mean_len, cfg.sigma, cfg.K_true, cfg.zipf_s, seed=seed)
    return w, d, n_docs


def host_cpu():
    """nproc and the CPU model of this host (lscpu, else /proc/cpuinfo)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    if model is None and os.path.exists("/proc/cpuinfo"):
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    return os.cpu_count() or 1, model


def time_oracle(cfg, target_tokens: int, iters: int, warmup: int = 0, omp: bool = False):
    """The CPU oracle as it stands on a bounded sample of the workload: tokens/s, tokens, docs,
    seconds, threads (omp: the OpenMP build over every host core; identical results)."""
    from oracle import oracle

    oracle.build(omp=omp)
    w, d, n_docs = oracle_sample(cfg, target_tokens)
    orc = oracle.OracleLDA(w, d, n_docs, cfg.V, cfg.K, seed=SAMPLER_SEED, omp=omp)
    if warmup:
        orc.iterate(warmup)
    t0 = time.perf_counter()
    orc.iterate(iters)
    dt = time.perf_counter() - t0
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)) if omp else 1
    return len(w) * iters / dt, len(w), n_docs, dt, threads


def arm_config(cfg, args, world: int) -> dict:
    """The workload both arms report (ours and --impl reference print the same dict)."""
    return {"workload": f"{cfg.name}-shaped synthetic LDA", "docs": cfg.n_docs, "V": cfg.V, "K": cfg.K,
            "mean_doc_len": cfg.mean_len, "doc_len_sigma": cfg.sigma, "alpha": cfg.alpha, "beta": cfg.beta,
            "g": args.g, "w_mode": args.w_mode, "split_threshold": args.split or 10000,
            "exact_draws": bool(args.exact_draws), "doc_block_kb": args.doc_block_kb or 32768,
            "sampler": "two-branch (ESCA)" if args.sampler == 2 else "three-branch",
            "schedule": ["per-iteration live items", "static item list", "no balancing"][args.schedule],
            "iterations_timed": [args.warmup + 1, args.warmup + args.steps],
            "parallelism": f"doc-partitioned x{world}",
            "l2": "inputs exceed L2 (corpus state "
                  f">{(int(cfg.n_docs * cfg.mean_len) * 12) >> 30} GiB vs 126 MB L2); no flush"}


def run_reference(args, rank, world=1):
    """--impl reference: the CPU oracle as it stands, on the host cores, on a bounded sample."""
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    tps, n, n_docs, dt, threads = time_oracle(cfg, args.ref_tokens, args.steps, args.warmup, omp=True)
    nproc, model = host_cpu()
    conf = arm_config(cfg, args, world)
    # the sample the oracle actually ran (same recipe, vocabulary, K and doc-length law)
    conf.update({"workload": f"{cfg.name}-shaped synthetic LDA, bounded oracle sample", "docs": n_docs,
                 "tokens_per_step": n})
    line = {
        "impl": "reference", "metric": METRIC, "value": tps, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": conf,
        "cpu_baseline": {"value": tps, "unit": UNIT, "cores": threads, "kind": "oracle", "nproc": nproc,
                         "cpu_model": model,
                         "sample": f"{n} tokens / {n_docs} docs of the {cfg.name}-shaped recipe (V={cfg.V}, "
                                   f"K={cfg.K}), iterations {args.warmup + 1}..{args.warmup + args.steps}, "
                                   f"C oracle OpenMP build on {threads} threads"},
        "e2e": {"value": tps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _fresh_nccl_id(world, rank, dist):
    """A ncclUniqueId bootstraps one communicator: every multi-rank handle needs a fresh one."""
    if world <= 1:
        return None
    from paper_2007_08725_b200 import lda

    obj = [lda.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="pubmed", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=2_000_000, help="oracle sample size for cpu_baseline")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--ref-tokens", type=int, default=1_000_000, help="oracle sample size per --impl reference step")
    ap.add_argument("--doc-block-kb", type=int, default=0,
                    help="sampler L2 tiling: KiB of D rows per doc window (0 = 32 MiB default, 4294967295 = off)")
    ap.add_argument("--curve-iters", type=int, default=100,
                    help="iterations of the paper-metric chain (mean tokens/s over 1..N, LLPT curve); 0 = skip")
    ap.add_argument("--llpt-every", type=int, default=10)
    # ablations (NEXT-3): W storage, S_est depth, large-word split, exact fp64 draws
    ap.add_argument("--w-mode", type=int, default=0, help="0 hybrid W (default), 1 all dense, 2 all sparse")
    ap.add_argument("--g", type=int, default=2, help="S_est depth g in {1,2,3} (Eq 10)")
    ap.add_argument("--split", type=int, default=0, help="large-word region size in tokens (0 = 10000)")
    ap.add_argument("--exact-draws", action="store_true", help="every sampled token on the exact fp64 path")
    ap.add_argument("--schedule", type=int, default=0, choices=[0, 1, 2],
                    help="sampler schedule: 0 per-iteration live items (default), 1 static list, 2 no balancing")
    ap.add_argument("--sampler", type=int, default=3, choices=[2, 3],
                    help="3: three-branch (default); 2: the paper's two-branch ESCA baseline mode (NEXT-1)")
    ap.add_argument("--ncu-traffic", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
    args = ap.parse_args()

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2007_08725_b200 import lda
    from paper_2007_08725_b200.synth import planted_corpus_torch

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lda.load()
    cfg = CONFIGS[args.config]

    # ---- corpus (same seed on every rank), doc partition, this rank's shard
    t_gen = time.perf_counter()
    w_all, d_all = planted_corpus_torch(cfg.n_docs, cfg.V, cfg.mean_len, cfg.sigma, cfg.K_true, cfg.zipf_s,
                                        seed=CORPUS_SEED, device=str(dev))
    L = torch.bincount(d_all, minlength=cfg.n_docs).cpu().numpy()
    bounds = lda.partition_docs(L, world)
    cum = np.concatenate([[0], np.cumsum(L)])
    doc_lo, doc_hi = bounds[rank], bounds[rank + 1]
    t0, t1 = int(cum[doc_lo]), int(cum[doc_hi])
    N_global = int(cum[-1])
    w = w_all[t0:t1].contiguous()
    d = (d_all[t0:t1] - doc_lo).contiguous()
    del w_all, d_all
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t_gen
    nccl_id = None
    if world > 1:
        obj = [lda.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.Stream(dev)  # a real stream (handle != 0): the library runs on it, events see it
    torch.cuda.set_stream(stream)
    t_create = time.perf_counter()
    knobs = dict(doc_block_kb=args.doc_block_kb, w_mode=args.w_mode, g=args.g, split_threshold=args.split,
                 exact_draws=args.exact_draws, sampler=args.sampler, schedule=args.schedule)
    ez = lda.EzLDA(w, d, doc_hi - doc_lo, cfg.V, cfg.K, seed=SAMPLER_SEED, rank=rank, world=world,
                   nccl_id=nccl_id, token_base=t0, stream=stream.cuda_stream, **knobs)
    torch.cuda.synchronize()
    create_s = time.perf_counter() - t_create

    # ---- warm-up, then exactly K timed steps bracketed by barrier + synchronize
    curve = []
    for _ in range(args.warmup):
        ez.iterate(1)
    torch.cuda.synchronize()
    ez.stats_sum(reset=True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            ez.iterate(1)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    S = ez.stats_sum(reset=True)
    llpt = ez.loglik()
    value = N_global * args.steps / (ms_max / 1e3)

    # ---- roofline of the dominant kernel (measured live: per-phase CUDA events on this stream)
    peak, peak_src = measured_peaks()
    # the sampler kernel's own CUDA-event time (the k_sampler launch; ms_sample also holds the
    # H4 item schedule and the n_k column sums)
    phases = {"sampler": (S.get("ms_sampler_kernel") or S["ms_sample"], S["model_bytes_sample"]),
              "doc_pass": (S["ms_docpass"], S["model_bytes_docpass"])}
    dom = max(phases, key=lambda k: phases[k][0])
    dom_ms, dom_bytes = phases[dom]
    achieved = (dom_bytes / args.steps) / (dom_ms / args.steps / 1e3) / 1e9 if dom_ms > 0 else 0.0
    traffic = None
    if os.path.exists(args.ncu_traffic):
        try:
            with open(args.ncu_traffic) as f:
                tj = json.load(f)
            traffic = tj.get(dom, {}).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "algorithmic_bytes_per_launch": dom_bytes / args.steps, "ms_per_launch": dom_ms / args.steps,
            "peak_source": peak_src,
            "whole_step": {"model_bytes_per_step": S["model_bytes"] / args.steps,
                           "achieved_gbs": S["model_bytes"] / (ms / 1e3) / 1e9,
                           "frac": S["model_bytes"] / (ms / 1e3) / 1e9 / peak}}

    if args.sampler == 2:  # the byte model describes the three-branch kernels
        roof.update({"achieved": None, "frac": None, "traffic": None, "algorithmic_bytes_per_launch": None,
                     "kernel": "two-branch draw + W rebuild",
                     "note": "two-branch baseline mode: no byte model; compare ms_per_step"})
        roof["whole_step"] = None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config(cfg, args, world),
        "tokens_per_step": N_global,
        "roofline": roof,
        "gpu_launches": int(S["kernel_launches"]),
        "phases_ms_per_step": {"wordprep": S["ms_wordprep"] / args.steps, "docpass": S["ms_docpass"] / args.steps,
                               "sample": S["ms_sample"] / args.steps, "allreduce": S["ms_allreduce"] / args.steps},
        "skip_S_frac": S["skip_S"] / max(S["n_tokens"], 1), "skip_final_frac": S["skip_final"] / max(S["n_tokens"], 1),
        "exact_redraw_frac": S["exact_redraws"] / max(S["sampled"], 1),
        "llpt_after": llpt, "setup_s": {"generate": gen_s, "create": create_s},
    }
    with_clk = clk.summary()
    line["clocks"] = with_clk
    del ez
    torch.cuda.synchronize()

    # ---- the paper's metric: mean tokens/s over iterations 1..100 and LLPT vs
    #      iteration (Eq 5), from a fresh chain (iteration times from the per-iteration events)
    if args.curve_iters:
        ezc = lda.EzLDA(w, d, doc_hi - doc_lo, cfg.V, cfg.K, seed=SAMPLER_SEED, rank=rank, world=world,
                        nccl_id=_fresh_nccl_id(world, rank, dist), token_base=t0, stream=stream.cuda_stream, **knobs)
        llpt_curve = [[0, ezc.loglik()]]
        ms_curve = []
        for it in range(1, args.curve_iters + 1):
            ezc.iterate(1)
            st = ezc.stats()
            ms_curve.append(round(st["ms_total"], 3))
            if it % args.llpt_every == 0 or it == args.curve_iters:
                llpt_curve.append([it, ezc.loglik()])
        del ezc
        msc = torch.tensor([sum(ms_curve)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(msc, op=dist.ReduceOp.MAX)
        line["paper_metric"] = {
            "what": f"mean sampled tokens/s over iterations 1..{args.curve_iters} of a fresh chain (P:1266), "
                    "per-iteration CUDA-event times (LLPT evaluations excluded)",
            "mean_tokens_per_s": N_global * args.curve_iters / (float(msc.item()) / 1e3),
            "ms_per_iteration": ms_curve, "llpt_vs_iteration": llpt_curve}

    # ---- end to end through the public API from pinned host buffers (create .. counts)
    if not args.no_e2e:
        hw = torch.empty(w.shape[0], dtype=torch.int32, pin_memory=True)
        hd = torch.empty(w.shape[0], dtype=torch.int32, pin_memory=True)
        hw.copy_(w)
        hd.copy_(d)
        hz = torch.empty(w.shape[0], dtype=torch.int16, pin_memory=True)
        del w, d
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        nccl_id2 = _fresh_nccl_id(world, rank, dist)
        if world > 1:
            dist.barrier()
        te = time.perf_counter()
        ez2 = lda.EzLDA(hw, hd, doc_hi - doc_lo, cfg.V, cfg.K, seed=SAMPLER_SEED, rank=rank, world=world,
                        nccl_id=nccl_id2, token_base=t0, stream=stream.cuda_stream, **knobs)
        ez2.iterate(args.warmup + args.steps)
        ez2.topics(out=hz)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - te
        if world > 1:
            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        del ez2
        nsteps = args.warmup + args.steps
        line["e2e"] = {"value": N_global * nsteps / e2e_s, "unit": UNIT,
                       "h2d_bytes_per_step": 8 * N_global / nsteps, "d2h_bytes_per_step": 2 * N_global / nsteps,
                       "what": f"ezlda_create from pinned host arrays (H2D) + {nsteps} iterations + topics D2H, "
                               "wall clock, setup included"}

    # ---- CPU oracle baseline (rank 0, N = 1 only): all host cores (OpenMP build) + one core
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nproc, model = host_cpu()
        tps, n, n_docs, dt, threads = time_oracle(cfg, args.cpu_tokens, args.cpu_iters, omp=True)
        tps1, n1, nd1, dt1, _ = time_oracle(cfg, args.cpu_tokens // 4, 1)
        line["cpu_baseline"] = {
            "value": tps, "unit": UNIT, "cores": threads, "kind": "oracle", "nproc": nproc, "cpu_model": model,
            "sample": f"{n} tokens / {n_docs} docs of the {cfg.name}-shaped recipe (V={cfg.V}, K={cfg.K}), "
                      f"iterations 1..{args.cpu_iters}, {dt:.1f} s, C oracle OpenMP build on {threads} threads",
            "single_thread": {"value": tps1, "unit": UNIT, "cores": 1,
                              "sample": f"{n1} tokens / {nd1} docs, iteration 1, {dt1:.1f} s"}}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

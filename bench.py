#!/usr/bin/env python
"""DynLP per-batch update benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c2|c1|c3|c4] [--points N]

A *step* is one engine.apply_batch (engine.py:328-413) over one batch of the
synthetic stream, all label columns (C2: 10 one-vs-rest columns).  The
stream is built with the make_stream rules (stream.py:56-183) from Gaussian
blobs and their cosine k-NN graph (builder.py:42-92 semantics), generated with
torch (fp64 GEMM + top-k) so that both bench arms build the identical stream
without the reference arm ever loading this repo's CUDA library.  Batches
before the warm-up window are a bootstrap (setup, untimed); the W warm-up
batches and the K timed batches are the last W+K batches of the stream
(|V| ~ 0.8M..1M at C2).

B200 arm (one process per GPU; N > 1 shards components over the ranks):
  value        device-resident batches (pre-uploaded), dlp_apply_batch_device
  e2e          host numpy batches through the public API (pinned staging + H2D
               inside each step, ingestion pipeline), report read back per step
  e2e_readback the e2e leg plus every label column read back to the host after
               each step (LabelState.F); its labels give the per-batch f digests
  cpu_baseline the compiled reference on the box's host cores for the first
               timed batch: every one-vs-rest column as its own reference run,
               the C runs concurrently (oracle/ref_workers.py), state hand-off
               of the GPU labels before the batch; the f bytes of every column
               are compared with the GPU's (sha256).
--impl reference: the compiled reference alone (rank 0), same machinery, on
the first min(K, --ref-steps) timed batches after 3 warm-up batches.  Its
state hand-off comes from baseline/handoff/ (written by this script's
--make-handoff on a B200, a file, never a library of this repo) or, failing
that, from the C restatement in oracle/ (port) replaying the stream.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]: 1M x 128, 10 classes, k=10, 1% seeds, 100 insert batches of 10k
    "c2": dict(n=1_000_000, dim=128, classes=10, k=10, seed_frac=0.01, batch=10_000,
               fractions=(0.99, 0.01, 0.0), seed=0, delta=1e-4,
               desc="C2: synthetic blobs 1M x 128-dim, 10 classes (one-vs-rest columns), "
                    "cosine kNN k=10, 1% seeds, 100 insert batches of 10k"),
    # C2 with binary labels (one label column): the single-column kernel path at 1M
    # (diagnostic; the reference itself is binary)
    "c2b": dict(n=1_000_000, dim=128, classes=2, k=10, seed_frac=0.01, batch=10_000,
                fractions=(0.99, 0.01, 0.0), seed=0, delta=1e-4,
                desc="C2 binary: synthetic blobs 1M x 128-dim, 2 classes (one label column), cosine kNN "
                     "k=10, 1% seeds, 100 insert batches of 10k"),
    # configs[0]: 10k x 16, 3 classes, k=10, 1% seeds, batches of 500
    "c1": dict(n=10_000, dim=16, classes=3, k=10, seed_frac=0.01, batch=500,
               fractions=(0.99, 0.01, 0.0), seed=0, delta=1e-4,
               desc="C1: synthetic blobs 10k x 16-dim, 3 classes, kNN k=10, 1% seeds, batches of 500"),
    # configs[3]: 10M x 64, k=16, 0.1% seeds (binary, one column), batches of 100k; the
    # working set (adjacency ~3.7 GB, labels 80 MB) is far beyond L2
    "c4": dict(n=10_000_000, dim=64, classes=2, k=16, seed_frac=0.001, batch=100_000,
               fractions=(0.99, 0.01, 0.0), seed=1, delta=1e-4,
               desc="C4: synthetic blobs 10M x 64-dim, binary, cosine kNN k=16, 0.1% seeds, "
                    "insert batches of 100k (single GPU)"),
    # configs[4] per SURVEY §8(d) D-2: 50M points uniform in the unit cube (one giant
    # component), exact 3-D k-NN k=10, binary (class = x > 1/2), 0.1% seeds; the
    # row-partitioned multi-GPU mode's workload (--shard-mode rows)
    "c5": dict(n=50_000_000, dim=3, classes=2, k=10, seed_frac=0.001, batch=500_000,
               fractions=(0.99, 0.01, 0.0), seed=2, delta=1e-4, gen="cube",
               desc="C5: 50M points uniform in [0,1]^3, exact 3-D kNN k=10 (single giant component), "
                    "binary, 0.1% seeds, insert batches of 500k"),
    # configs[2] per SURVEY §8(d) D-2: a 1.7M-point dataset; phase 1 = 100 insert batches
    # of 10k (|V| -> 1M, untimed), phase 2 = 100 mixed batches of 6.9k unlabeled + 0.1k
    # GT inserts + 3k deletes (|V| 1.0M -> 1.4M alive ... the timed tail)
    "c3": dict(n=1_700_000, dim=128, classes=10, k=10, seed_frac=0.01, batch=10_000,
               fractions=(0.69, 0.01, 0.30), seed=0, delta=1e-4, boot_batches=100, mixed_batches=100,
               desc="C3: blobs 1.7M x 128, 10 classes, kNN k=10; 100 insert batches of 10k "
                    "(|V| -> 1M), then 100 mixed batches 69/1/30 insert/gt/delete of 10k"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def stream_key(cfg):
    key = "_".join(str(cfg[k]) for k in ("n", "dim", "classes", "k", "seed_frac", "batch", "seed")) + \
        "_" + "_".join(str(x) for x in cfg["fractions"])
    if cfg.get("boot_batches"):
        key += f"_b{cfg['boot_batches']}m{cfg['mixed_batches']}"
    if cfg.get("gen"):
        key += "_" + cfg["gen"]
    return key + "_knn64"


def load_stream_npz(path):
    from paper_2604_06596_b200.batch import BatchUpdate

    z = np.load(path)
    # every z[...] access re-reads the whole array: load each one once (slicing a
    # fresh full copy per batch kept ~100 copies alive)
    a = {k: z[k] for k in ("ids", "gt", "own", "oth", "w", "dels", "io", "eo", "do", "classes")}
    io, eo, do = a["io"], a["eo"], a["do"]
    batches = [BatchUpdate(t=t, insert_ids=a["ids"][io[t]:io[t + 1]], insert_gt=a["gt"][io[t]:io[t + 1]],
                           edge_owner=a["own"][eo[t]:eo[t + 1]], edge_other=a["oth"][eo[t]:eo[t + 1]],
                           edge_w=a["w"][eo[t]:eo[t + 1]], deletes=a["dels"][do[t]:do[t + 1]])
               for t in range(len(io) - 1)]
    return batches, a["classes"]


def make_stream(cfg, device):
    """(batches, classes, cache path, stream sha256).  The k-NN graph comes from
    torch (fp64, GPU when present): input generation shared by both arms."""
    from paper_2604_06596_b200 import streams

    cache_dir = os.environ.get("DYNLP_BENCH_CACHE", "/tmp/dynlp_bench_cache")
    os.makedirs(cache_dir, exist_ok=True)
    path = os.path.join(cache_dir, f"stream_{stream_key(cfg)}.npz")
    if not os.path.exists(path):
        t0 = time.time()
        if cfg.get("gen") == "cube":
            bl = streams.uniform_cube(cfg["n"], cfg["seed"])
            edges = streams.knn_graph_grid3d(bl.x, cfg["k"])
        else:
            bl = streams.make_blobs(cfg["n"], cfg["dim"], cfg["classes"], cfg["seed"])
            if cfg["n"] > 2_000_000 and device:
                # 10M+ points: this repo's tensor-core k-NN (exact edge set; a torch fp64
                # GEMM + top-k would need 8n bytes per query row).  Only the B200 arm
                # runs these configs (no CPU reference at this size).
                from paper_2604_06596_b200.knn import FeatureMatrix, knn_graph

                edges = knn_graph(FeatureMatrix(bl.x), cfg["k"], device=int(device.split(":")[-1]))
            else:
                edges = streams.knn_graph_torch64(bl.x, cfg["k"], device=device or "cpu")
        gt = streams.stratified_seeds(bl.classes, cfg["seed_frac"], cfg["seed"])
        fi, fg, fd = cfg["fractions"]
        phases = None
        if fd > 0:  # phase 1 grows the graph with inserts, phase 2 is mixed
            phases = [(cfg["boot_batches"], cfg["batch"], 0.99, 0.01, 0.0),
                      (cfg["mixed_batches"], cfg["batch"], fi, fg, fd)]
        s = streams.phased_stream(cfg["n"], edges, bl.classes, gt, cfg["batch"], cfg["seed"], fi, fg, fd,
                                  initial_gt=2 * cfg["classes"], phases=phases)
        log(f"[bench] stream built in {time.time() - t0:.1f}s: {len(s.batches)} batches, {len(edges)} kNN edges")
        b = s.batches
        tmp = path + f".tmp{os.getpid()}.npz"
        np.savez(tmp, ids=np.concatenate([x.insert_ids for x in b]), gt=np.concatenate([x.insert_gt for x in b]),
                 own=np.concatenate([x.edge_owner for x in b]), oth=np.concatenate([x.edge_other for x in b]),
                 w=np.concatenate([x.edge_w for x in b]), dels=np.concatenate([x.deletes for x in b]),
                 io=np.cumsum([0] + [len(x.insert_ids) for x in b]),
                 eo=np.cumsum([0] + [len(x.edge_owner) for x in b]),
                 do=np.cumsum([0] + [len(x.deletes) for x in b]), classes=s.classes)
        os.replace(tmp, path)
    batches, classes = load_stream_npz(path)
    z = np.load(path)
    h = hashlib.sha256()
    for k in ("ids", "gt", "own", "oth", "w", "dels"):
        h.update(np.ascontiguousarray(z[k]).tobytes())
    return batches, classes, path, h.hexdigest()


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            # nvidia-smi's start-up (NVML init) stalls the device for tens of ms:
            # let it finish before the timed region begins
            t_end = time.time() + 5.0
            while not self.lines and time.time() < t_end:
                time.sleep(0.05)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def handoff_dir():
    return os.path.join(ROOT, "baseline", "handoff")


def handoff_path(cfg, t_h):
    return os.path.join(handoff_dir(), f"{stream_key(cfg)}_t{t_h}.npz")


def f_digests(F):
    """sha256 of every label column's bytes (fp64, slots 0..n-1)."""
    from oracle.ref_workers import f_digest

    return [f_digest(F[c]) for c in range(F.shape[0])]


def ref_digest_cache(cfg):
    d = os.environ.get("DYNLP_BENCH_CACHE", "/tmp/dynlp_bench_cache")
    return os.path.join(d, f"refdigests_{stream_key(cfg)}.json")


def run_ref_pool(stream_path, ncol, t_h, F_h, delta, batches_to_run, n_timed, threads):
    """C concurrent reference column runs from the hand-off labels F_h (state
    before batch t_h): apply `batches_to_run` in order, time the last
    n_timed.  Returns (per-step seconds, per-step column reports, per-step
    digests {t: [...]}, column seconds of the timed steps)."""
    from oracle.ref_workers import RefColumnPool

    cache_dir = os.environ.get("DYNLP_BENCH_CACHE", "/tmp/dynlp_bench_cache")
    hpath = os.path.join(cache_dir, f"handoff_{os.getpid()}_t{t_h}.npy")
    if F_h is not None:
        np.save(hpath, np.ascontiguousarray(F_h))
    pool = RefColumnPool(stream_path, ncol, t_h, hpath, delta, threads)
    try:
        times, reps, digs = [], [], {}
        for i, t in enumerate(batches_to_run):
            s = time.time()
            dt, rep, dg, _ = pool.step(t)
            timed = i >= len(batches_to_run) - n_timed
            log(f"[bench] reference batch t={t}: {dt:.2f}s (slowest column), wall {time.time() - s:.2f}s"
                f"{'' if timed else ' (warm-up)'}")
            if timed:
                times.append(dt)
                reps.append(rep)
            digs[int(t)] = dg
        return times, reps, digs
    finally:
        pool.close()
        try:
            os.remove(hpath)
        except OSError:
            pass


def port_handoff(batches, t_h, ncol, delta, threads):
    """State before batch t_h by the C restatement (oracle/, the 'port'),
    columns in parallel: the fallback when no hand-off file exists."""
    from oracle import OracleEngine
    from oracle.ref_workers import column_gt  # noqa: F401  (same remap rule)

    orc = OracleEngine(max(2, ncol if ncol > 1 else 2), threads=threads)
    s = time.time()
    for b in batches[:t_h]:
        orc.apply_batch(b, delta=delta)
    log(f"[bench] port hand-off: {t_h} batches replayed in {time.time() - s:.1f}s")
    f, _ = orc.labels()
    return np.ascontiguousarray(f.reshape(ncol, -1)[:, :orc.num_slots])


def reference_arm(args, cfg, batches, spath, ssha, world):
    T = len(batches)
    K, W = args.steps, args.warmup
    ncol = 1 if cfg["classes"] <= 2 else cfg["classes"]
    t0 = T - K
    k_ref = max(1, min(K, args.ref_steps))
    w_ref = max(1, min(W, 3))
    t_h = t0 - w_ref
    cores = host_cores()
    threads = max(1, cores // ncol)
    hp = handoff_path(cfg, t_h)
    F_h, source = None, None
    if os.path.exists(hp):
        z = np.load(hp)
        if str(z["stream_sha"]) == ssha and int(z["t_h"]) == t_h:
            F_h, source = np.ascontiguousarray(z["F"]), f"file {os.path.relpath(hp, ROOT)} (B200 arm --make-handoff)"
        else:
            log(f"[bench] hand-off {hp} does not match this stream; falling back to the port")
    if F_h is None:
        F_h, source = port_handoff(batches, t_h, ncol, cfg["delta"], cores), "oracle/ C restatement (port) replay"
    run = list(range(t_h, t0 + k_ref))
    times, reps, digs = run_ref_pool(spath, ncol, t_h, F_h, cfg["delta"], run, k_ref, threads)
    val = 1e3 * float(np.mean(times))
    try:
        with open(ref_digest_cache(cfg), "w") as fh:
            json.dump({"stream_sha": ssha, "digests": digs}, fh)
    except OSError:
        pass
    timed = f"t={t0}..{t0 + k_ref - 1}"
    line = {"impl": "reference", "metric": "dynlp_ms_per_batch", "value": val, "unit": "ms/batch",
            "n_gpus": world, "steps": k_ref, "steps_requested": K, "warmup": w_ref,
            "ms_per_step": val, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "points": cfg["n"], "timed_batches": timed,
                       "label_columns": ncol, "delta": cfg["delta"]},
            "cpu_baseline": {"value": val, "unit": "ms/batch", "cores": ncol * threads if ncol > 1 else threads,
                             "kind": "reference",
                             "sample": f"batches {timed} of the B200 arm's timed window (first {k_ref} of {K}), "
                                       f"all {ncol} one-vs-rest columns, each an unmodified compiled-reference "
                                       f"apply_batch in its own process (EngineConfig(threads={threads})), the "
                                       f"columns concurrently on {cores} host cores; step = slowest column; "
                                       f"warm-up batches t={t_h}..{t0 - 1}; state before t={t_h} from {source}",
                             "cpu_model": cpu_model(), "host_cores": cores},
            "e2e": {"value": val, "unit": "ms/batch", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "column_reports": reps,
            "f_sha256": {str(t): hashlib.sha256("".join(d).encode()).hexdigest()[:16] for t, d in digs.items()},
            "stream_sha256": ssha[:16]}
    print(json.dumps(line), flush=True)


def make_handoff(args, cfg, batches, ssha, device_index):
    """B200 arm utility: the labels before batch t_h = T - K - min(W, 3) (the
    reference arm's hand-off point) written as a compressed .npz."""
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch

    T = len(batches)
    t_h = T - args.steps - max(1, min(args.warmup, 3))
    g, lab = DynamicGraph(device_index, num_classes=max(2, cfg["classes"])), LabelState()
    g.reserve(sum(len(b.insert_ids) for b in batches), sum(len(b.edge_owner) for b in batches))
    ecfg = EngineConfig(delta=cfg["delta"])
    for b in batches[:t_h]:
        lab, _ = apply_batch(g, lab, b, ecfg)
    F = np.ascontiguousarray(lab.F)
    g.close()
    out = args.handoff_out or handoff_path(cfg, t_h)
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    np.savez_compressed(out, F=F, t_h=t_h, stream_sha=ssha)
    log(f"[bench] hand-off t_h={t_h} ({F.shape}) -> {out} ({os.path.getsize(out) / 1e6:.1f} MB)")


def knn_leg(cfg, device_index, K):
    """Per-batch k-NN edge construction: the arriving points
    of a batch queried against all N points, on tensor cores."""
    from paper_2604_06596_b200 import streams
    from paper_2604_06596_b200.knn import KnnIndex

    bl = streams.make_blobs(cfg["n"], cfg["dim"], cfg["classes"], cfg["seed"])
    idx = KnnIndex(bl.x, device_index)
    q = cfg["batch"]
    runs = []
    for r in range(max(3, min(K, 5)) + 1):
        q0 = cfg["n"] - q * (r % 3 + 1)
        s = time.perf_counter()
        idx.query(q0, q0 + q, cfg["k"])
        wall = (time.perf_counter() - s) * 1e3
        st = idx.stats()
        if r:  # first call is a warm-up
            runs.append((wall, st.screen_ms, st.recheck_ms, st.exact_ms, st.fallback_queries))
    idx.close()
    wall, scr, rec, ex, fb = (float(np.median([x[i] for x in runs])) for i in range(5))
    kext = 3 * ((cfg["dim"] + 15) // 16 * 16)  # three Dp-deep fp16 products per pair
    flops_alg = 2.0 * q * cfg["n"] * cfg["dim"]
    flops_exec = 2.0 * q * cfg["n"] * kext
    peak = measured_tensor_peak()
    alg = flops_alg / (scr * 1e-3) / 1e12
    return {"queries": q, "points": cfg["n"], "dim": cfg["dim"], "k": cfg["k"],
            "ms": wall, "screen_ms": scr, "recheck_ms": rec, "exact_fallback_ms": ex,
            "fallback_queries": fb, "pairs_per_s": q * cfg["n"] / (wall * 1e-3),
            "roofline": {"bound": "tensor", "achieved": alg, "peak": peak, "unit": "TFLOP/s",
                         "frac": alg / peak, "executed_tflops": flops_exec / (scr * 1e-3) / 1e12,
                         "note": "achieved = algorithmic 2QND per screen launch time; executed = 3 fp16 "
                                 "products (hi/lo split) per pair; peak = MEASURED_PEAKS.json bf16_tflops "
                                 "(dense fp16 == bf16 rate)",
                         "kernel": "k_knn_screen (tcgen05.mma kind::f16, TMEM accumulators)"}}


def measured_tensor_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["bf16_tflops"])
    return 1590.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def traffic_record(config):
    p = os.path.join(ROOT, "profiles", "lp_kernel_traffic.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d.get(config) if isinstance(d.get(config), dict) else (d if config == "c2" else None)
        except Exception:
            return None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--points", "--n", dest="n", type=int, default=None,
                    help="override point count (smaller smoke runs; --points under torchrun)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-knn", action="store_true", help="skip the k-NN edge-construction leg")
    ap.add_argument("--no-itlp", action="store_true", help="skip the ItLP comparison leg")
    ap.add_argument("--no-readback", action="store_true", help="skip the e2e label read-back leg")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of sharding")
    ap.add_argument("--shard-mode", default="components", choices=["components", "rows", "components_hash"],
                    help="N > 1: shard connected components, or partition rows (giant component)")
    ap.add_argument("--ref-steps", type=int, default=5, help="reference arm: timed batches (bounded sample)")
    ap.add_argument("--make-handoff", action="store_true",
                    help="write the reference arm's hand-off labels (B200 engine) and exit")
    ap.add_argument("--handoff-out", default=None)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = dict(CONFIGS[args.config])
    if args.n:
        cfg["n"] = args.n

    import torch

    have_gpu = torch.cuda.is_available()
    dist = None
    if world > 1:
        import torch.distributed as dist

        # DYNLP_BENCH_BACKEND=gloo + DYNLP_BENCH_ONE_DEVICE=1: exercise the multi-rank
        # path with every rank on GPU 0 (protocol checks on a one-GPU box)
        dist.init_process_group(os.environ.get("DYNLP_BENCH_BACKEND", "nccl" if have_gpu else "gloo"))
    if args.impl == "reference" and rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    if os.environ.get("DYNLP_BENCH_ONE_DEVICE"):
        local = 0
    device = f"cuda:{local}" if have_gpu else None
    if have_gpu:
        torch.cuda.set_device(local)

    batches, classes, spath, ssha = make_stream(cfg, device)
    if have_gpu:
        torch.cuda.empty_cache()
    T = len(batches)
    K, W = args.steps, args.warmup
    t0 = T - K  # first timed batch
    tw = t0 - W  # first warm-up batch
    if tw < 1:
        raise SystemExit(f"stream has {T} batches; need more than steps+warmup")
    ncol = 1 if cfg["classes"] <= 2 else cfg["classes"]
    delta = cfg["delta"]

    if args.impl == "reference":
        reference_arm(args, cfg, batches, spath, ssha, world)
        if dist:
            dist.destroy_process_group()
        return
    if args.make_handoff:
        make_handoff(args, cfg, batches, ssha, local)
        return

    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch

    ecfg = EngineConfig(delta=delta)

    # N > 1: one stream, connected components sharded over the ranks
    # (sharded.py; phase bookkeeping reduced with NCCL); --replicas runs N
    # independent copies instead.
    sharded = world > 1 and not args.replicas
    # over NCCL the engines run every exchange on their own communicator (device
    # buffers, no Python in the loop); gloo (CPU protocol checks) uses the host
    # collective.  DYNLP_BENCH_HOST_COLLECTIVE=1 forces the host path.
    nccl = sharded and dist.get_backend() == "nccl" and not os.environ.get("DYNLP_BENCH_HOST_COLLECTIVE")
    if sharded:
        from paper_2604_06596_b200.sharded import (ShardedGraph, apply_batch_sharded, nccl_unique_id,
                                                   torch_collective)

        coll = None if nccl else torch_collective(device=device if dist.get_backend() == "nccl" else None)

    def new_graph():
        if sharded:
            if nccl:  # a fresh communicator per engine (the id travels over the process group)
                obj = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                g = ShardedGraph(local, max(2, cfg["classes"]), rank, world, None, args.shard_mode, nccl_id=obj[0])
            else:
                g = ShardedGraph(local, max(2, cfg["classes"]), rank, world, coll, args.shard_mode)
            return g, LabelState()
        return DynamicGraph(local, num_classes=max(2, cfg["classes"])), LabelState()

    def step(g, lab, b):
        if sharded:
            return apply_batch_sharded(g, lab, b, ecfg)
        return apply_batch(g, lab, b, ecfg)

    boot_reports = []

    def bootstrap(record=False):
        g, lab = new_graph()
        # capacity hint for the whole stream (setup, untimed): no reallocation in timed steps
        g.reserve(sum(len(b.insert_ids) for b in batches), sum(len(b.edge_owner) for b in batches))
        s = time.time()
        for b in batches[:t0]:
            lab, r = step(g, lab, b)
            if record:
                boot_reports.append(r if isinstance(r, list) else [r])
        log(f"[bench] rank {rank}: bootstrap+warmup {t0} batches in {time.time() - s:.1f}s, |V|={g.num_slots}")
        return g, lab

    # ---------------- B200 arm -----------------------------------------------------
    gA, labA = bootstrap(record=True)
    # the reference on the host cores: bounded samples only (a replay of the
    # reference's structure at 10M+ points alone takes longer than the bench)
    cpu_ok = cfg["n"] <= 2_000_000
    F0 = np.ascontiguousarray(labA.F) if rank == 0 and not args.no_cpu_baseline and not sharded and cpu_ok else None
    # device-resident batches for the value leg
    dev = []
    for b in batches[t0:]:
        dev.append(dict(t=b.t, n_ins=len(b.insert_ids), n_edges=len(b.edge_owner), n_del=len(b.deletes),
                        insert_ids=torch.as_tensor(np.asarray(b.insert_ids, np.int64), device=device),
                        insert_gt=torch.as_tensor(np.asarray(b.insert_gt, np.int8), device=device),
                        edge_owner=torch.as_tensor(np.asarray(b.edge_owner, np.int64), device=device),
                        edge_other=torch.as_tensor(np.asarray(b.edge_other, np.int64), device=device),
                        edge_w=torch.as_tensor(np.asarray(b.edge_w, np.float64), device=device),
                        deletes=torch.as_tensor(np.asarray(b.deletes, np.int64), device=device)))
    torch.cuda.synchronize()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    # ---- value leg: inputs resident in HBM --------------------------------------
    barrier()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    repsA = []
    for s in range(K):
        if sharded:  # sharded batches enter through the host path on every rank
            r = step(gA, labA, batches[t0 + s])[1]
            repsA.append(r if isinstance(r, list) else [r])
        else:
            repsA.append(gA.apply_device(dev[s], ecfg, trusted=True))
    ev1.record()
    barrier()
    clk = clocks.stop()
    ms_value = max_over_ranks(ev0.elapsed_time(ev1)) / K
    gA.close()

    # ---- e2e leg: host buffers through the public API ---------------------------
    tb = batches[t0:]
    h2d = sum(b.insert_ids.nbytes + b.insert_gt.nbytes + b.edge_owner.nbytes + b.edge_other.nbytes +
              b.edge_w.nbytes + b.deletes.nbytes for b in tb) // K
    from paper_2604_06596_b200 import _native
    import ctypes

    rep_bytes = ctypes.sizeof(_native.Report) * ncol

    def e2e_leg(readback):
        g, lab = bootstrap()
        barrier()
        ev0.record()
        reps, Fs = [], []
        for i, b in enumerate(tb):
            if sharded:
                lab, r = step(g, lab, b)
            else:  # ingestion pipeline: batch i+1 is validated and copied while batch i runs
                lab, r = apply_batch(g, lab, b, ecfg, next_batch=tb[i + 1] if i + 1 < len(tb) else None)
            if readback:
                Fs.append(lab.F)  # every label column, read back from HBM
            reps.append(r if isinstance(r, list) else [r])
        ev1.record()
        barrier()
        ms = max_over_ranks(ev0.elapsed_time(ev1)) / K
        n_last = g.num_slots
        g.close()
        return ms, reps, Fs, n_last

    ms_e2e, repsB, _, _ = e2e_leg(False)
    readback = None
    gpu_digests = {}
    if not args.no_readback and not sharded:
        ms_rb, repsR, Fs, _ = e2e_leg(True)
        for i, F in enumerate(Fs):
            gpu_digests[t0 + i] = f_digests(F)
        rb_bytes = sum(F.nbytes for F in Fs) // K
        readback = {"value": ms_rb, "unit": "ms/batch", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(rb_bytes + rep_bytes),
                    "note": "e2e plus every label column (LabelState.F, fp64) read back to the host after "
                            "each step"}
        del Fs

    # ---- aggregates -------------------------------------------------------------
    upd = sum(r.updates for step_ in repsA for r in step_)
    edges = sum(r.edges_traversed for step_ in repsA for r in step_)
    lp_ms = sum(step_[0].lp_kernel_ms for step_ in repsA)  # one fused launch per step
    launches = sum(step_[0].gpu_launches for step_ in repsA) / K
    rounds = sum(step_[0].lp_rounds for step_ in repsA) / K
    urows = sum(step_[0].lp_union_rows for step_ in repsA)
    uent = sum(step_[0].lp_union_entries for step_ in repsA)
    # algorithmic bytes of the fused kernel: per union row
    # 16 B row bounds + 4 B emask; per gathered entry 4 B id + 8 B weight + 8*C B
    # label vector; per (vertex, column) update 8 B f read + 8 B staged write +
    # 8 B staged read + 8 B commit write.
    alg_bytes = 20.0 * urows + (12.0 + 8.0 * ncol) * uent + 32.0 * upd
    achieved = alg_bytes / (lp_ms * 1e-3) / 1e9 if lp_ms > 0 and uent > 0 else None
    survey_bytes = 32.0 * upd + 21.0 * edges  # SURVEY §8(d) D-4 per-column model
    peak, peak_kind = measured_peaks()
    tr = traffic_record(args.config) if not args.n else None
    same = all(a[c].iterations == b[c].iterations and a[c].updates == b[c].updates
               for a, b in zip(repsA, repsB) for c in range(len(a)))
    ingest_edges = sum(len(b.edge_owner) + len(b.deletes) for b in tb)
    boot_ms = [r[0].wall_time_ms for r in boot_reports]
    line = {
        "metric": "dynlp_ms_per_batch", "value": ms_value, "unit": "ms/batch", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms_value, "higher_is_better": False,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "points": cfg["n"], "timed_batches": f"t={t0}..{T - 1}",
                   "label_columns": ncol, "delta": delta,
                   "parallelism": ((f"component-sharded x{world} ({'LPT' if args.shard_mode == 'components' else 'hash'}"
                                    f" placement, " if args.shard_mode != "rows" else
                                    f"row-partitioned x{world} (per-round all-gather of packed rows, ")
                                   + ("NCCL in the engine)" if nccl else "host collective)")
                                   if sharded else f"replicas x{world}"),
                   "l2": "no flush: each batch's working set (adjacency pool, edge log, label and staging "
                         "columns) exceeds the 126 MB L2"},
        "edges_per_s": edges / (ms_value * K * 1e-3),
        "ingest_edges_per_s": ingest_edges / (ms_e2e * K * 1e-3),
        "vertex_updates_per_batch": upd / K, "edge_relaxations_per_batch": edges / K,
        "all_batches": {"batches": len(boot_ms) + K, "mean_ms": float(np.mean(boot_ms + [r[0].wall_time_ms
                                                                                           for r in repsA])),
                        "tail10_mean_ms": float(np.mean([r[0].wall_time_ms for r in repsA][-10:])),
                        "note": "host wall time per apply_batch over the whole stream (bootstrap batches "
                                "included, device batches for the timed tail)"},
        "lp_kernel_share": lp_ms / (ms_value * K),
        "lp_rounds_per_batch": rounds, "lp_union_rows_per_batch": urows / K,
        "lp_union_entries_per_batch": uent / K,
        "survey_model_gbs": survey_bytes / (lp_ms * 1e-3) / 1e9 if lp_ms > 0 else None,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": (tr or {}).get("dram_bytes_per_launch"),
                     "traffic_note": "DRAM read+write bytes of one k_lp_fused launch of this config from an ncu "
                                     "--set full capture (profiles/lp_kernel_traffic.json); compare with "
                                     "algorithmic_bytes_per_launch",
                     "algorithmic_bytes_per_launch": alg_bytes / K if uent > 0 else None,
                     "kernel": "k_lp_fused (persistent frontier/certify loop)",
                     "algorithmic_bytes": "fused kernel: 20 B/union row + (12 + 8C) B/gathered entry + "
                                          "32 B/(vertex, column) update; see DESIGN.md",
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
        "e2e": {"value": ms_e2e, "unit": "ms/batch", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(rep_bytes)},
        "gpu_launches": launches, "clocks": clk,
        "step_wall_ms": {"value": [round(r[0].wall_time_ms, 2) for r in repsA],
                         "e2e": [round(r[0].wall_time_ms, 2) for r in repsB],
                         "lp_kernel": [round(r[0].lp_kernel_ms, 2) for r in repsA]},
        "certify_sweeps_per_batch": sum(r.certify_sweeps for step_ in repsA for r in step_) / K,
        "legs_identical_work": same,
        "stream_sha256": ssha[:16],
    }
    if readback:
        line["e2e_readback"] = readback
        line["f_sha256"] = {str(t): hashlib.sha256("".join(d).encode()).hexdigest()[:16]
                            for t, d in gpu_digests.items()}
        rc = ref_digest_cache(cfg)
        if os.path.exists(rc):  # the reference arm ran first on this box
            try:
                rd = json.load(open(rc))
                if rd.get("stream_sha") == ssha:
                    common = [int(t) for t in rd["digests"] if int(t) in gpu_digests]
                    line["parity_with_reference_arm"] = {
                        "batches": common, "columns": ncol,
                        "f_bytes_equal": all(rd["digests"][str(t)] == gpu_digests[t] for t in common)}
            except Exception as e:
                log(f"[bench] reference digests unreadable: {e!r}")
    if rank == 0 and not args.no_itlp and not sharded:
        # the paper's comparison: ItLP (full sweeps, baselines.py:236-253)
        # on the same first timed batch from the same state, on the B200
        from paper_2604_06596_b200.engine import itlp_batch_solve

        gC, labC = bootstrap()
        s_ = time.perf_counter()
        _, repI = itlp_batch_solve(gC, labC, batches[t0], ecfg)
        wall_itlp = (time.perf_counter() - s_) * 1e3
        repI = repI if isinstance(repI, list) else [repI]
        gC.close()
        line["itlp"] = {"ms": wall_itlp, "lp_kernel_ms": repI[0].lp_kernel_ms,
                        "sweeps_per_column": [r.iterations for r in repI],
                        "updates": sum(r.updates for r in repI),
                        "dynlp_ms_same_batch": repsA[0][0].wall_time_ms,
                        "speedup_dynlp_vs_itlp": wall_itlp / max(repsA[0][0].wall_time_ms, 1e-9)}
    if rank == 0 and not args.no_knn and not cfg.get("gen"):  # cosine k-NN leg (blob configs)
        line["knn"] = knn_leg(cfg, local, K)
    if rank == 0 and F0 is None and not cpu_ok and not args.no_cpu_baseline:
        line["cpu_baseline"] = {"skipped": f"{cfg['n']} points: the reference's structure replay alone exceeds a "
                                           "bounded sample; C2 (1M) carries the CPU baseline"}
    if rank == 0 and F0 is not None:
        cores = host_cores()
        threads = max(1, cores // ncol)
        times, reps, digs = run_ref_pool(spath, ncol, t0, F0, delta, [t0], 1, threads)
        cpu_ms = 1e3 * times[0]
        gpu_rep = [(r.iterations, r.updates, r.max_change, int(r.converged)) for r in repsA[0]]
        line["cpu_baseline"] = {
            "value": cpu_ms, "unit": "ms/batch", "cores": ncol * threads if ncol > 1 else threads,
            "kind": "reference",
            "sample": f"batch t={t0}, all {ncol} one-vs-rest columns, each an unmodified compiled-reference "
                      f"apply_batch in its own process (EngineConfig(threads={threads})), columns concurrently "
                      f"on {cores} host cores (step = slowest column); state hand-off of the GPU labels "
                      f"before t={t0}",
            "cpu_model": cpu_model(), "host_cores": cores,
            "parity_with_gpu": {"reports_equal": [tuple(x) for x in reps[0]] == gpu_rep,
                                "f_bytes_equal": (digs[t0] == gpu_digests[t0]) if t0 in gpu_digests else None,
                                "columns": ncol},
            "speedup_vs_value": cpu_ms / ms_value, "speedup_vs_e2e": cpu_ms / ms_e2e}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

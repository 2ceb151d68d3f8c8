"""Benchmark of the hot path: one step = one iteration of Alg. 5
on the config-2 geometry (BASELINE.json configs[2], the headline roofline
config): forward g = A f, ratio y/(g + r), backward b2 = A^T ratio, closed-form
update -- every stage a libcacsi kernel called through the C ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]

Metric (BASELINE.json): forward+backward pairs/s (2 * N_vox * N_det voxel-pixel
pairs per step), with voxel-pixel-energy terms/s and the roofline fraction of
the dominant kernel reported beside it.  Multi-GPU: the path does not shard
(north_star: one GPU, no collectives) -> N independent replicas, value =
all ranks' pairs / max-over-ranks time, scaling "weak".

At N=1 the config-2 line also carries "config3" (BASELINE configs[3]: 50 EM
iterations with setup, final relative error, OSEM-64) and "config4" (BASELINE
configs[4], energy-resolving: this script with --config 4 in a child process).

--impl reference times the fp64 CPU oracle (the reference arm of this tier) on
a bounded sample of the same workload, on this box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import make_config  # noqa: E402
from workloads.configs import seeded_rng  # noqa: E402

METRIC = "forward+backward pairs/s"
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="cacsi", choices=["cacsi", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--options", default=None, help="kernel-variant options (cacsi_geometry_create_ex)")
    ap.add_argument("--no-config3", action="store_true", help="skip the config-3 reconstruction key")
    ap.add_argument("--no-config4", action="store_true", help="skip the config-4 (energy-resolving) key")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0, help="target seconds of oracle work")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        loaded = [s for s in sm if mx and s > 0.3 * max(mx)] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------- replicas (N>1) --
def max_over_ranks(ms: float, world: int, device=None) -> float:
    """Timed-region duration of the job = max over ranks (the path does not
    shard: N independent replicas)."""
    if world <= 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank_step: float, steps: int, world: int, total_ms: float) -> float:
    """Whole-job value: units all ranks processed / max-over-ranks time."""
    return units_per_rank_step * steps * world / (total_ms / 1e3)


# ------------------------------------------------------------ work counts --
def work_counts(cfg):
    """Pairs and nominal terms per operator application."""
    pairs = cfg.n_vox * cfg.n_det
    return pairs, pairs * cfg.ne


# ---------------------------------------------------------------- GPU arm --
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1603_06400_b200 as P

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    cfg = make_config(args.config)
    d = cfg.desc()
    G0 = P.Geometry(d, device=local)
    # synthetic Poisson data of the config-3 recipe on this geometry (input only)
    f_true = torch.as_tensor(cfg.f).to(dev)
    l_true = torch.empty(G0.g_shape, dtype=torch.float32, device=dev)
    G0.forward(f_true, l_true)
    torch.cuda.synchronize()
    lt = l_true.double().cpu().numpy()
    s = 1e4 / lt.mean()
    y_np = seeded_rng(cfg.seed, 2).poisson(s * lt + 5.0).astype(np.float32)
    r_np = np.full(G0.g_shape, 5.0, np.float32)
    G0.close()
    d["scale"] = s
    # geometry setup, timed over three creations (the median is reported): a creation right
    # after another handle freed its ~6 GB varies with the driver's reclaim of that memory
    setup_runs, stage_runs = [], []
    for i in range(3):
        torch.cuda.synchronize()
        t_setup = time.perf_counter()
        G = P.Geometry(d, device=local, options=args.options)  # host tables, ESAI tables, bitmaps, pair cache
        torch.cuda.synchronize()
        setup_runs.append((time.perf_counter() - t_setup) * 1e3)
        stage_runs.append({k[len("setup_us_"):]: G.query(k) / 1e3 for k in (
            "setup_us_tables", "setup_us_bitmaps", "setup_us_bound", "setup_us_pc_fill", "setup_us_pc_perm",
            "setup_us_pc_segwin", "setup_us_host", "setup_us_total")})
        if i < 2:
            G.close()
    med = sorted(range(3), key=lambda i: setup_runs[i])[1]
    setup_ms, setup_stages = setup_runs[med], stage_runs[med]
    y = torch.as_tensor(y_np).to(dev)
    r = torch.as_tensor(r_np).to(dev)
    ones = torch.ones(G.g_shape, dtype=torch.float32, device=dev)
    b1 = torch.empty(G.f_shape, dtype=torch.float32, device=dev)
    G.backward(ones, b1)
    torch.cuda.synchronize()
    f0 = float((y_np - r_np).sum() / b1.double().sum().item())
    f = torch.full(G.f_shape, f0, dtype=torch.float32, device=dev)
    l = torch.empty(G.g_shape, dtype=torch.float32, device=dev)
    b2 = torch.empty(G.f_shape, dtype=torch.float32, device=dev)
    fn = torch.empty(G.f_shape, dtype=torch.float32, device=dev)
    beta = 1e-3
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    launches_per_step = [0]

    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device=dev)

    def step(ev=None):
        """One Alg. 5 iteration through cacsi_iterate (on ESAI handles the ratio and max|w|
        ride in the forward's final partial sum and the update in the backward's)."""
        if ev:
            ev[0].record(stream)
        G.iterate(f, y, r, b1, beta, 1, ws)
        if ev:
            ev[1].record(stream)
        launches_per_step[0] = G.last_launch_count

    def op_step(ev):
        """The same iteration as separate operator calls (forward, ratio, backward,
        update): the per-operator split reported beside the step."""
        ev[0].record(stream)
        G.forward(f, l)
        ev[1].record(stream)
        G.ratio(l, y, r, l)
        ev[2].record(stream)
        G.backward(l, b2)
        ev[3].record(stream)
        G.update(f, b1, b2, beta, fn)
        f.copy_(fn)
        ev[4].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [[E() for _ in range(2)] for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(float(i))  # L2 flush between timed steps (outside the events)
        step(evs[i])
    torch.cuda.synchronize()
    ck = clocks.stop()
    launches_timed = launches_per_step[0]  # (step() is reused below on the comparison handle)
    t_step = [e[0].elapsed_time(e[1]) for e in evs]
    # per-kernel times (CUDA events around every libcacsi kernel, same stream) in a
    # separate pass, so the timed steps above carry no per-kernel events
    n_aux = max(1, min(args.steps, 5))
    G.kernel_times()   # discard
    G.set_timing(True)
    for i in range(n_aux):
        flush.fill_(float(i))
        step()
    torch.cuda.synchronize()
    G.set_timing(False)
    ktimes = G.kernel_times()
    # per-operator split (unfused calls)
    evo = [[E() for _ in range(5)] for _ in range(n_aux)]
    for i in range(n_aux):
        flush.fill_(float(i))
        op_step(evo[i])
    torch.cuda.synchronize()
    t_fwd = [e[0].elapsed_time(e[1]) for e in evo]
    t_bwd = [e[2].elapsed_time(e[3]) for e in evo]
    t_opstep = [e[0].elapsed_time(e[4]) for e in evo]
    total_ms = max_over_ranks(float(sum(t_step)), world, dev)
    ms_per_step = total_ms / args.steps
    pairs, nominal_terms = work_counts(cfg)
    value = job_throughput(2 * pairs, args.steps, world, total_ms)

    # ---- e2e: the same step through the host-buffer C ABI (pinned buffers)
    fh = torch.full(G.f_shape, f0, dtype=torch.float32).pin_memory().numpy()
    yh = torch.as_tensor(y_np).pin_memory().numpy()
    rh = torch.as_tensor(r_np).pin_memory().numpy()
    b1h = b1.cpu().pin_memory().numpy()
    G.iterate_host(fh, yh, rh, b1h, beta, 1)  # warm the staging buffers
    e2e_ms = []
    for i in range(max(1, min(args.steps, 5))):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G.iterate_host(fh, yh, rh, b1h, beta, 1)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_value = 2 * pairs * world / (np.mean(e2e_ms) / 1e3)
    h2d = (fh.nbytes + yh.nbytes + rh.nbytes + b1h.nbytes)
    d2h = fh.nbytes

    # ---- the same step without the pair cache (geometry and breakpoint location
    # recomputed per pair inside the operators, CACSI_PAIR_CACHE=0), for comparison
    on_the_fly = None
    if G.query("pair_cache_records") > 0:
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        G2 = P.Geometry(d, device=local, options="pair_cache=0")
        torch.cuda.synchronize()
        setup2_ms = (time.perf_counter() - t2) * 1e3
        G, Gc = G2, G
        f.fill_(f0)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        ev2 = [[E() for _ in range(2)] for _ in range(max(1, min(args.steps, 5)))]
        for i, ev in enumerate(ev2):
            flush.fill_(float(i))
            step(ev)
        torch.cuda.synchronize()
        ms2 = float(np.mean([e[0].elapsed_time(e[1]) for e in ev2]))
        on_the_fly = {"ms_per_step": ms2, "value": 2 * pairs / (ms2 / 1e3), "setup_ms": setup2_ms,
                      "amortized_ms_per_step_50": (setup2_ms + 50 * ms2) / 50,
                      "note": "option pair_cache=0: pair geometry and breakpoint location recomputed per pair per call"}
        G.close()
        G = Gc

    # ---- roofline: the dominant operator call, work per
    # SURVEY.md §8(d)'s per-unit figures (FP32 lane-ops: 4 per effective term
    # forward, 6 backward, 60 per open pair geometry, 12 per pair mask test)
    mf, mb = float(np.mean(t_fwd)), float(np.mean(t_bwd))
    counts = json.load(open(os.path.join(ROOT, "workloads", "work_counts.json")))[str(cfg.seed)]
    nb_bp = G.query("esai_breakpoints")
    kern = {k: {"avg_ms": v[0] / v[1], "launches": v[1]} for k, v in ktimes.items()}
    fwd_k = [k for k in kern if k in ("k_pad_rows", "k_tc_pack_a", "k_tc_gemm_W", "k_esai_fwd", "k_esai_fwd_ts", "k_pc_fwd",
                                      "k_sum_parts_f64", "k_forward", "k_sum_f64", "k_forward_er", "k_sum_f32",
                                      "k_er_tab", "k_er_fwd")]
    bwd_k = [k for k in kern if k in ("k_absmax", "k_esai_bwd", "k_pc_bwd", "k_tc_gemm_b2", "k_sum_parts_f32",
                                      "k_backward", "k_transpose", "k_backward_er", "k_er_absmax", "k_er_bwd",
                                      "k_er_bsum")]
    op_ms = {"cacsi_forward": sum(kern[k]["avg_ms"] for k in fwd_k),
             "cacsi_backward": sum(kern[k]["avg_ms"] for k in bwd_k)}
    dom = max(op_ms, key=op_ms.get)
    ops = survey_ops(dom, counts)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    peak = sms * 128 * 1965e6 / 1e12  # FP32 lane-ops/s at the max SM clock
    achieved = ops / (op_ms[dom] / 1e3) / 1e12
    kdom = max(kern, key=lambda k: kern[k]["avg_ms"] * kern[k]["launches"])
    kflops = alg_flops(kdom, cfg, counts, nb_bp)
    roofline = {"bound": "alu", "kernel": dom + " (" + " + ".join(fwd_k if dom == "cacsi_forward" else bwd_k) + ")",
                "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": "Tops/s", "frac": round(achieved / peak, 4),
                "traffic": None, "algorithmic_ops_per_launch": ops, "avg_launch_ms": op_ms[dom],
                "peak_note": f"{sms} SMs x 128 FP32 lanes x 1965 MHz (max clock) lane-ops/s, derived (DESIGN.md §8); "
                             "work = SURVEY §8(d) per-unit figures x exact counts (workloads/work_counts.json)",
                "kernel_level": {"kernel": kdom, "avg_ms": kern[kdom]["avg_ms"], "alg_flops": kflops,
                                 "tflops": round(kflops / (kern[kdom]["avg_ms"] / 1e3) / 1e12, 3),
                                 "frac_of_74.4_tflops": round(kflops / (kern[kdom]["avg_ms"] / 1e3) / 1e12 /
                                                               (2 * peak), 4)}}
    if ck.get("sm_mhz"):
        roofline["frac_at_observed_clock"] = round(achieved / (peak * ck["sm_mhz"] / 1965.0), 4)
    # DRAM traffic of the operator's kernels from the committed ncu --set full capture
    # (profiles/r2k_dram_traffic.json, bytes per launch); kernels it does not list are omitted
    # (profiles/r2s4_er_dram_traffic.json for the energy-resolving kernels of config 4)
    try:
        er = bool(cfg.energy_resolving)
        fn = "r2s4_er_dram_traffic.json" if er else "r2k_dram_traffic.json"
        tr = json.load(open(os.path.join(ROOT, "profiles", fn)))["kernels"]
        ks = [k for k in (fwd_k if dom == "cacsi_forward" else bwd_k) if k in tr]
        if ks:
            roofline["traffic"] = float(sum(tr[k]["dram_read_bytes"] + tr[k]["dram_write_bytes"] for k in ks))
            roofline["traffic_note"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch of " + " + ".join(ks) + \
                f" (profiles/{fn}); " + ("the operator's open-pair records (16 B per pair forward, 12 B backward) "
                                         "read once" if er else
                                         "compulsory bytes of the operator (f, g, w, b, tables) are ~0.1 GB -- "
                                         "the rest is the W / A scratch of the ESAI contraction")
    except Exception:
        pass
    eff = counts["effective_terms"]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    # HBM roofline of the dominant pair-cache kernel: algorithmic bytes
    # per launch = the record bytes per open pair (P, packed (b, tau), pixel q: 10 B on
    # config 2, read once) + the 8-byte list offsets
    # + the operator's table it gathers from once (k_pc_fwd: the W rows,
    # n_vox x ldw x 4 B; k_pc_bwd: w, n_det x 4 B, and the A rows it writes,
    # n_vox x ldw x 4 B), against the measured copy bandwidth
    roofline_hbm = None
    kpc = [k for k in ("k_pc_fwd", "k_pc_bwd") if k in kern]
    if kpc:
        kd = max(kpc, key=lambda k: kern[k]["avg_ms"])
        ldw = G.query("esai_ldw")
        nrec = G.query("pair_cache_padded_records")  # records streamed, padding included
        tab = cfg.n_vox * ldw * 4 if kd == "k_pc_fwd" else cfg.n_det * 4 + cfg.n_vox * ldw * 4
        rb = G.query("pair_cache_record_bytes")
        bytes_ = float(rb) * nrec + 8.0 * cfg.n_vox * cfg.det_nx + tab + float(G.query("pair_cache_window_base_bytes"))
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        ach = bytes_ / (kern[kd]["avg_ms"] / 1e3) / 1e9
        roofline_hbm = {"bound": "hbm", "kernel": kd, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "traffic": None, "algorithmic_bytes_per_launch": bytes_,
                        "avg_launch_ms": kern[kd]["avg_ms"],
                        "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in peaks else
                        "fallback 6650 GB/s (B200_PROFILING.md)",
                        "bytes_note": f"{rb} B per record (pair cache, incl. padding) + 2 B per 128-record window "
                                      "(pixel bases) + list offsets + the gathered table once (DESIGN.md §8)"}
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "r2q8_dram_traffic.json")))["kernels"]
            if kd in tr:
                roofline_hbm["traffic"] = tr[kd]["dram_read_bytes"] + tr[kd]["dram_write_bytes"]
        except Exception:
            pass

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "n_vox": cfg.n_vox, "n_det": cfg.n_det, "nq": cfg.nq, "ne": cfg.ne,
                   "step": "Alg.5 iteration through cacsi_iterate: forward (+ ratio, max|w| in its final sum), "
                           "backward (+ update in its final sum), beta=1e-3",
                   "pairs_per_step": 2 * pairs, "l2": "flushed (256 MB write) between timed steps",
                   "parallelism": f"replicas x{world}"},
        "forward_ms": mf, "backward_ms": mb, "operator_calls_ms_per_step": float(np.mean(t_opstep)),
        "operator_split_note": "forward_ms / backward_ms: cacsi_forward / cacsi_backward as separate calls "
                               "(with cacsi_ratio and cacsi_update between them), CUDA events, separate pass",
        "forward_pairs_per_s": pairs / (mf / 1e3), "backward_pairs_per_s": pairs / (mb / 1e3),
        "nominal_terms_per_s": 2 * nominal_terms * world / (ms_per_step / 1e3),
        "effective_terms_per_s": 2 * float(eff) * world / (ms_per_step / 1e3),
        "gpu_launches": launches_timed * args.steps,
        "kernels": kern, "esai_breakpoints": nb_bp, "ts_rho": G.query("ts_rho"),
        "clocks": ck, "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": float(np.mean(e2e_ms))},
        "peaks_source": "MEASURED_PEAKS.json" if peaks else "fallback",
        "setup_ms": setup_ms, "setup_stages_ms": setup_stages, "setup_ms_runs": [round(x, 2) for x in setup_runs],
        "amortized_ms_per_step_50": (setup_ms + 50 * ms_per_step) / 50,
        "amortized_note": "(geometry setup + 50 timed-rate steps) / 50: Alg. 5 runs T iterations on one geometry "
                          "(PAPER.md:363-377); the pair cache is built once per geometry (PAPER.md:236-241)",
        "pair_cache_records": G.query("pair_cache_records"),
        "on_the_fly": on_the_fly,
    }
    if roofline_hbm is not None:
        # the dominant kernels stream the pair cache: HBM is their roof; the SURVEY
        # FP32 accounting of the whole operator is kept beside it
        out["roofline_alu_survey"] = out["roofline"]
        out["roofline"] = roofline_hbm
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_sample_s)
    if rank == 0 and args.config == 2 and not args.no_config3:
        G.close()
        out["config3"] = run_config3(P, torch, dev, local)
    if rank == 0 and world == 1 and args.config == 2 and not args.no_config4:
        out["config4"] = run_config4()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    G.close()
    if rank == 0:
        print(json.dumps(out), flush=True)


CONFIG4_KEYS = ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "config", "forward_ms", "backward_ms",
                "effective_terms_per_s", "gpu_launches", "clocks", "roofline", "e2e", "setup_ms",
                "amortized_ms_per_step_50")


def run_config4(steps=3, warmup=3, timeout_s=900):
    """BASELINE.json configs[4] (energy-resolving, the regime SURVEY §8 calls the stress case)
    measured in the default bench run, so the driver's line carries it: this script with
    --config 4 in a child process (its own CUDA context and memory; the config-2 handle
    is closed), the same timing rules (warm-up, L2 flush, CUDA events, clocks, e2e through
    cacsi_iterate_host); the child's cpu_baseline is skipped (the config-4 oracle sample is
    in profiles/r2s5a_bench4.json)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--config", "4", "--steps", str(steps), "--warmup", str(warmup),
           "--no-cpu-baseline"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, env=dict(os.environ))
        line = [x for x in r.stdout.strip().splitlines() if x.startswith("{")]
        if r.returncode != 0 or not line:
            return {"error": f"rc={r.returncode}: {(r.stderr or '').strip().splitlines()[-1:]}"}
        d = json.loads(line[-1])
        return {k: d[k] for k in CONFIG4_KEYS if k in d}
    except Exception as ex:  # reported, never hidden: the key then says why it is missing
        return {"error": repr(ex)}


def run_config3(P, torch, dev, local, n_iter=50, osem_outer=3):
    """BASELINE.json configs[3] on the device: config-1 geometry, Poisson data with mean
    count 1e4 + background 5, beta = 1e-3, uniform start; 50 iterations of Alg. 5
     through ONE cacsi_iterate call, setup included in the
    time-to-solution; relative error of f^50 against f_true; and Alg. 6 with the
    paper's 64 symmetric subsets (rho_x = 8, rho_y = 16).  CUDA
    events on the launching stream; every stage a libcacsi kernel."""
    cfg = make_config(1)
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    stream = torch.cuda.current_stream()
    G0 = P.Geometry(cfg.desc(), device=local)
    f_true = torch.as_tensor(cfg.f).to(dev)
    l_true = torch.empty(G0.g_shape, dtype=torch.float32, device=dev)
    G0.forward(f_true, l_true)
    torch.cuda.synchronize()
    lt = l_true.double().cpu().numpy()
    G0.close()
    s = 1e4 / lt.mean()
    y_np = seeded_rng(3, 2).poisson(s * lt + 5.0).astype(np.float32)
    d = cfg.desc()
    d["scale"] = s
    y = torch.as_tensor(y_np).to(dev)
    r = torch.full(y.shape, 5.0, dtype=torch.float32, device=dev)
    beta = 1e-3
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G = P.Geometry(d, device=local)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    ones = torch.ones(G.g_shape, dtype=torch.float32, device=dev)
    b1 = torch.empty(G.f_shape, dtype=torch.float32, device=dev)
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device=dev)
    jout = torch.zeros(1, dtype=torch.float64, device=dev)
    eb = [E(), E()]
    eb[0].record(stream)
    G.backward(ones, b1)
    eb[1].record(stream)
    torch.cuda.synchronize()
    f0 = float((y_np - 5.0).sum() / b1.double().sum().item())
    f = torch.full(G.f_shape, f0, dtype=torch.float32, device=dev)
    G.iterate(f, y, r, b1, beta, 1, ws)  # warm-up (allocator pools, clocks)
    f.fill_(f0)
    G.neg_loglik(f, y, r, beta, jout, ws)
    j0 = jout.item()
    ei = [E(), E()]
    ei[0].record(stream)
    G.iterate(f, y, r, b1, beta, n_iter, ws)
    ei[1].record(stream)
    torch.cuda.synchronize()
    G.neg_loglik(f, y, r, beta, jout, ws)
    j50 = jout.item()
    ft = f_true.double()
    rel = float(torch.linalg.norm(f.double() - ft) / torch.linalg.norm(ft))
    em_ms = ei[0].elapsed_time(ei[1])
    # Alg. 6, 64 subsets
    sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, 8, 16).ravel()
    nsub = int(sub.max()) + 1
    lists = [np.flatnonzero(sub == p).astype(np.int32) for p in range(nsub)]
    offs = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int32)
    allpix = torch.as_tensor(np.concatenate(lists)).to(dev)
    b1s = torch.empty((nsub,) + G.f_shape, dtype=torch.float32, device=dev)
    for p in range(nsub):
        G.backward_subset(ones, allpix[offs[p]:offs[p + 1]], b1s[p])
    fo = torch.full(G.f_shape, f0, dtype=torch.float32, device=dev)
    G.osem(fo, y, r, b1s, allpix, offs, beta, None, 1, ws)  # capture the outer-iteration graph
    fo.fill_(f0)
    eo = [[E(), E()] for _ in range(osem_outer)]
    for a, b in eo:
        a.record(stream)
        G.osem(fo, y, r, b1s, allpix, offs, beta, None, 1, ws)
        b.record(stream)
    torch.cuda.synchronize()
    G.neg_loglik(fo, y, r, beta, jout, ws)
    jo = jout.item()
    out = {"workload": "config3: config-1 geometry, y ~ Poisson(s A f_true + 5) with mean count 1e4, r = 5, "
                       "beta = 1e-3 (quadratic, 4-neighbour), uniform f0 = sum(y - r) / sum(b1)",
           "setup_ms": setup_ms, "b1_ms": eb[0].elapsed_time(eb[1]),
           "em_iters": n_iter, "em_ms_total": em_ms, "em_ms_per_iter": em_ms / n_iter,
           "time_to_solution_ms": setup_ms + eb[0].elapsed_time(eb[1]) + em_ms,
           "objective_J0": j0, "objective_J50": j50, "final_rel_err_vs_f_true": rel,
           "rel_err_note": "an ill-posed problem (262,144 unknowns, 16,384 measurements): the error is not a target",
           "osem_subsets": nsub, "osem_ms_per_outer_iter": float(np.median([a.elapsed_time(b) for a, b in eo])),
           "osem_objective_after_outer": jo, "osem_outer_iters": osem_outer,
           "osem_beats_50_em": bool(jo <= j50)}
    G.close()
    return out


def survey_ops(op, counts):
    """SURVEY.md §8(d) algorithmic work of one operator application, in FP32
    lane-ops: forward 4 / backward 6 per effective term, geometry 60 per open
    pair, mask test 12 per pair."""
    per_term = 4 if op == "cacsi_forward" else 6
    return float(per_term * counts["effective_terms"] + 60 * counts["open_pairs"] + 12 * counts["pairs"])


def alg_flops(kernel, cfg, counts, nb):
    """Algorithmic FP32 flops (FMA = 2) of one launch of a libcacsi kernel on
    this workload (DESIGN.md §8 table): the minimal arithmetic of the formulas
    the kernel evaluates, times the units it processes."""
    pairs, open_ = counts["pairs"], counts["open_pairs"]
    gemm = 2.0 * cfg.n_vox * nb * cfg.nq
    table = {
        "k_tc_gemm_W": gemm,                           # W = F S~^T (tensor cores, 3xTF32: 3 MMAs per product)
        "k_tc_gemm_b2": gemm,                          # b2 = A S~
        "k_esai_fwd": 2 * pairs + (46 + 11) * open_,   # bit pop, pair geometry, locate + lerp + accumulate
        # TS: footprint shared; per open pair the source-side terms (r^, G_so: 9), the r^-dependent
        # geometry (23), locate (6) and lerp + accumulate (4)
        "k_esai_fwd_ts": 2 * pairs + (9 + 23 + 10) * open_,
        "k_esai_bwd": 2 * pairs + (46 + 6 + 6) * open_,  # compaction, geometry, locate, fixed-point deposits
        "k_pc_fwd": 4 * open_,                         # pair cache: a0 W_b + a1 W_b+1 accumulated (2 FFMA)
        "k_pc_bwd": 6 * open_,                         # pair cache: w scale, two weighted deposits
        "k_forward": 10 * pairs + 46 * open_ + 7 * counts["effective_terms"],
        "k_backward": 10 * pairs + 46 * open_ + 9 * counts["effective_terms"],
        # energy-resolving per-term kernels: per effective term 4 flops forward (hat lerp 2 +
        # accumulate 2), 6 backward (weight 2 + two deposits 4); geometry per open pair
        "k_forward_er": 10 * pairs + 46 * open_ + 4 * counts["effective_terms"],
        "k_backward_er": 10 * pairs + 46 * open_ + 6 * counts["effective_terms"],
        "k_er_fwd": 4 * counts["effective_terms"],
        "k_er_bwd": 6 * counts["effective_terms"],
    }
    return float(table.get(kernel, 0.0))


# --------------------------------------------------------- CPU (oracle) arm --
def _oracle_sample(cfg, budget_s):
    """Time the oracle's forward on a pixel sample and backward on a voxel sample,
    sized to ~budget_s seconds on this host's cores.  Returns (pairs, seconds, desc)."""
    import oracle
    O = oracle.Geometry(cfg)
    f = cfg.f.astype(np.float64)
    w = np.ones(O.g_shape)
    rng = np.random.default_rng(0)
    # calibrate on a tiny sample
    pix = rng.choice(cfg.n_det, 64, replace=False)
    t0 = time.perf_counter()
    O.forward_pixels(f, pix)
    per_pix = (time.perf_counter() - t0) / 64
    npix = int(max(64, min(cfg.n_det, 0.5 * budget_s / max(per_pix, 1e-9))))
    vox_cost = per_pix * cfg.n_det / cfg.n_vox
    nvox = int(max(8, min(cfg.n_vox, 0.5 * budget_s / max(vox_cost, 1e-9))))
    pix = rng.choice(cfg.n_det, npix, replace=False)
    vox = rng.choice(cfg.n_vox, nvox, replace=False)
    t0 = time.perf_counter()
    O.forward_pixels(f, pix)
    t1 = time.perf_counter()
    O.backward_voxels(w, vox)
    t2 = time.perf_counter()
    pairs = npix * cfg.n_vox + nvox * cfg.n_det
    return pairs, t2 - t0, f"forward on {npix} random pixels x all {cfg.n_vox} voxels + backward on {nvox} " \
                          f"random voxels x all {cfg.n_det} pixels of {cfg.name} ({t1 - t0:.1f}s + {t2 - t1:.1f}s)"


def cpu_baseline(cfg, budget_s):
    pairs, secs, desc = _oracle_sample(cfg, budget_s)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": pairs / secs, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    cfg = make_config(args.config)
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        _oracle_sample(cfg, budget)
    tot_pairs, tot_s, desc = 0, 0.0, ""
    for _ in range(args.steps):
        p, s, desc = _oracle_sample(cfg, budget)
        tot_pairs += p
        tot_s += s
    value = tot_pairs / tot_s
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg.name, "n_vox": cfg.n_vox, "n_det": cfg.n_det, "nq": cfg.nq, "ne": cfg.ne},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_gpu(a)

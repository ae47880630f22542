"""Benchmark: B0 -> J/psi K pi phase-space generation + weight integration
(BASELINE.json configs[1]: 1e8 events per B200), plus the FCN (configs[3]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = generate EVENTS_PER_GPU events per GPU into HBM (13 fp64 SoA
columns, 104 B/event), with the weight moments (sum w, sum w^2) fused into the
same kernel, then the fold of each rank's partials into its 1024 super-chunk
records, the cross-GPU gather of those records (NCCL) and the deterministic
fold -> weight sum / mean / variance.  Weak scaling: rank r generates the
global rows of its super-chunks (parallel.shard_range), ~EVENTS_PER_GPU each.

Prints ONE JSON line on rank 0: the C2 headline with its roofline (copy and
live write-only HBM), e2e through pinned host columns, clocks, the CPU
baseline (the bit-exact C port, and the reference's own Python from
baseline/_ref on C1-C5 and the FCN), the FCN (plain nll(), session, batched,
fit), and the other configs.  `--impl reference` times the reference
algorithm's CPU implementation (the bit-exact C oracle port, all host
threads) on the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "phase-space events/s (B0→J/ψKπ, fp64) and FCN evals/s @1e7 evts, 1–8 B200"
M_B0, DAUGHTERS = 5.27966, (3.0969, 0.493677, 0.13957039)
EVENTS_PER_GPU = 100_000_000
BYTES_PER_EVENT = 8 * (4 * 3 + 1)          # algorithmic HBM bytes written per 3-body event
FCN_EVENTS = 10_000_000
WORKLOAD = "C2: B0->J/psi K pi phase-space generation + weight sum/mean/variance, 1e8 events/GPU in HBM"


def _peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json copy BW)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def _traffic() -> float | None:
    """dram read+write bytes per launch of the generator, from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "generate_traffic.json")) as fh:
            return float(json.load(fh)["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


def _fp64_roofline(kernel: str, events_per_s_per_gpu: float, note: str = "") -> dict | None:
    """FP64-pipe roofline of an FP64-bound kernel (C4 FCN, C5 fused integration;
    SURVEY.md 8(d)): the live per-GPU event rate x the kernel's DP instructions
    per event (ncu, committed) against the DFMA instruction rate measured by
    tools/fp64_peak.cu (committed; MEASURED_PEAKS.json has no FP64 figure)."""
    d = None
    for tag in ("r02", "r01"):   # the newest committed DP-count capture
        try:
            with open(os.path.join(ROOT, "profiles", f"{tag}_fp64_roofline.json")) as fh:
                d = json.load(fh)
            k, pk = d["kernels"][kernel], d["peak"]
            break
        except (OSError, KeyError, ValueError):
            d = None
    if d is None:
        return None
    inst = events_per_s_per_gpu * k["dp_inst_per_event"]
    return {"bound": "fp64", "achieved": inst * 1e-12, "peak": pk["dp_inst_per_s"] * 1e-12,
            "unit": "T DP inst/s", "frac": inst / pk["dp_inst_per_s"], "dp_inst_per_event": k["dp_inst_per_event"],
            "frac_ncu_one_launch": k.get("dp_inst_frac_of_peak_ncu"),
            **({"note": note} if note else {})}


class NvmlClockSampler:
    """SM clock + clock-event reasons polled through NVML every ~0.5 ms in a
    thread for exactly the timed region (the region is tens of ms, shorter
    than nvidia-smi's sampling period).  Falls back to nvidia-smi."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.ok = False

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            visible = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(visible.split(",")[self.gpu]) if visible else self.gpu
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi fallback
            self.fallback = ClockSampler(self.gpu).__enter__()
            return self
        self.stop = threading.Event()

        def poll():
            nv, h = self.nv, self.h
            power = 0.0
            k = 0
            while not self.stop.is_set():
                try:
                    if k % 8 == 0:      # power is the slow query: every 8th sample
                        power = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                    self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                         nv.nvmlDeviceGetCurrentClocksEventReasons(h), power))
                except Exception:  # noqa: BLE001
                    pass
                k += 1
                time.sleep(0.0005)

        # the timed loop only enqueues work and then waits: a short GIL
        # switch interval lets the poller run while the main thread holds it
        import sys
        self.switch = sys.getswitchinterval()
        sys.setswitchinterval(1e-4)
        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        while not self.samples and self.thread.is_alive():   # first sample before the region
            time.sleep(0.0002)
        return self

    def __exit__(self, *exc):
        if not self.ok:
            return self.fallback.__exit__(*exc)
        self.stop.set()
        self.thread.join(timeout=5)
        import sys
        sys.setswitchinterval(self.switch)

    def summary(self) -> dict:
        if not self.ok:
            return self.fallback.summary()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "source": "nvml"}
        mhz = [s[0] for s in self.samples]
        active = sorted({n for _, r, _ in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(mhz), "sm_min_mhz": min(mhz), "sm_max_mhz": self.max_mhz,
                "power_w_max": max(s[2] for s in self.samples), "samples": len(self.samples),
                "reasons": active, "source": "nvml, ~0.5 ms polling inside the timed region"}


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=10)

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit()),
                "samples": len(rows), "reasons": reasons}


def bench_config(events_per_gpu: int, events_per_step: int) -> dict:
    """The workload both arms run (identical dicts for the same --gpus)."""
    return {"workload": WORKLOAD, "events_per_gpu": events_per_gpu, "events_per_step": events_per_step,
            "decay": "B0(5.27966) -> J/psi(3.0969) K(0.493677) pi(0.13957039), mother at rest, RngKey(1,1)",
            "rng": "reference SplitMix64 stream (bit-exact to the reference)",
            "l2": "each step writes 104 B/event (10.4 GB per GPU >> 126 MB L2): no flush needed"}


def _best_of(fn, reps: int) -> float:
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def _reference_python():
    """The reference package itself, installed offline into baseline/_ref
    (`pip install --no-index --no-deps --target baseline/_ref /root/reference/pkg`;
    git-ignored, travels to the GPU box with the snapshot).  None when absent."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "hepkit")):
        return None
    if path not in sys.path:
        sys.path.append(path)      # appended: never shadows the drop-in package
    try:
        import hepkit
    except Exception:  # noqa: BLE001 -- a broken install is reported as absent
        return None
    return hepkit


def cpu_reference(reps: int = 3) -> dict:
    """CPU baseline of C2 (generation + weight sum / mean / variance) on this
    box's host cores: best-of-`reps` wall clock at 1
    thread and at os.cpu_count() threads, for
      * the reference's own Python (`hepkit.phsp_generate(..., workers=w)` +
        numpy weight sums) from baseline/_ref, when installed;
      * the bit-exact C port of the same algorithm (oracle/, -ffp-contract=off,
        pthreads) -- the headline `value` (the faster of the two CPU paths).
    Bounded samples (rates, not the full 1e8): ~10-30 s of CPU work in all."""
    import numpy as np

    from oracle import oracle as O  # the CPU baseline leg (test/bench infrastructure only)

    cores = os.cpu_count() or 1

    def port(n, threads):
        def run():
            w = O.generate(DAUGHTERS, M_B0, n, 1, 1, threads=threads)["weight"]
            return float(np.sum(w)), float(np.sum(w * w))
        return n / _best_of(run, reps)

    out = {"unit": "events/s", "cores": cores, "kind": "port", "best_of": reps}
    n_port = 50_000_000 if cores >= 8 else 10_000_000
    out["value"] = port(n_port, cores)
    out["port_1_thread"] = port(5_000_000, 1)
    ref = _reference_python()
    rp = None
    if ref is not None:
        spec, mother = ref.DecaySpec(M_B0, DAUGHTERS), ref.FourVector.at_rest(M_B0)
        rp = {"source": "baseline/_ref hepkit (the unmodified reference)", "events": 1_000_000}
        for workers in (1, cores):
            def run(workers=workers):
                blk = ref.phsp_generate(spec, mother, 1_000_000, ref.RngKey(1, 1), workers=workers)
                w = np.asarray(blk.column("weight"))
                return float(np.sum(w)), float(np.sum(w * w))
            rp[f"workers_{workers}"] = 1_000_000 / _best_of(run, reps)
    if ref is not None:
        rp["fcn_1e7"] = reference_fcn(ref, cores, reps)
        rp.update(reference_configs(ref, cores, reps))
    out["reference_python"] = rp if rp else "baseline/_ref not installed on this box"
    out["sample"] = (f"C2 rate: port {n_port} events at {cores} threads and 5e6 at 1 thread; reference Python "
                     f"1e6 events at workers=1 and {cores}; reference FCN at 1e7 events; best of {reps}")
    return out


def reference_configs(ref, cores: int, reps: int) -> dict:
    """The reference's own Python on the other BASELINE configs (SURVEY
    8(d) CPU baseline), rates in events/s at workers=1 and all cores, best of
    `reps`: C1 (1e5 events per phsp_generate call), C3 (phsp_generate +
    phsp_decay_chain J/psi -> mu mu, 1e6 events), C5 (phsp_average of m12^2
    over a stored 1e6-event block)."""
    spec, mother = ref.DecaySpec(M_B0, DAUGHTERS), ref.FourVector.at_rest(M_B0)
    sub = ref.DecaySpec(3.0969, (0.1056583755, 0.1056583755))
    blk = ref.phsp_generate(spec, mother, 1_000_000, ref.RngKey(1, 1))

    def m12(cols):
        e = cols["p1_e"] + cols["p2_e"]
        px = cols["p1_px"] + cols["p2_px"]
        py = cols["p1_py"] + cols["p2_py"]
        pz = cols["p1_pz"] + cols["p2_pz"]
        return (e * e - px * px - py * py - pz * pz,)

    runs = {
        "C1": (100_000, lambda w: ref.phsp_generate(spec, mother, 100_000, ref.RngKey(1, 1), workers=w)),
        "C3": (1_000_000, lambda w: ref.phsp_decay_chain(
            ref.phsp_generate(spec, mother, 1_000_000, ref.RngKey(1, 1), workers=w), 1, sub, ref.RngKey(2, 1),
            workers=w)),
        "C5": (1_000_000, lambda w: ref.phsp_average(ref.identity(), blk, m12, workers=w)),
    }
    out = {}
    for name, (n, fn) in runs.items():
        out[name] = {"events": n, "unit": "events/s"}
        for workers in (1, cores):
            out[name][f"workers_{workers}"] = n / _best_of(lambda w=workers, f=fn: f(w), reps)
    return out


def reference_fcn(ref, cores: int, reps: int) -> dict:
    """The reference's own FCN (hepkit.nll, fitting.py:175-210) on this box's
    host cores at the C4 size: the benchmark model (4e6 Gaussian + 6e6
    exponential on [0, 10]) over 1e7 events, parameters alternating as in our
    arm's loop (norms recomputed), best of `reps` at workers=1 and all cores."""
    import numpy as np
    P = ref.Parameter
    region = ref.BoundedRegion(((0.0, 10.0),))
    mean, sigma, tau = P("mean", 5.0), P("sigma", 0.5), P("tau", 3.0)
    g = ref.shape_gaussian(mean, sigma)
    e = ref.shape_exponential(tau)
    model = ref.add_pdfs([P("n_sig", 4e6), P("n_bkg", 6e6)],
                         [ref.make_pdf(g, ref.gaussian_norm(g), region),
                          ref.make_pdf(e, ref.exponential_norm(e), region)])
    rs = np.random.default_rng(7)
    x = np.clip(np.concatenate([rs.normal(5.0, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
    store = ref.ColumnStore.from_columns(ref.ColumnSchema.real64("x0"), [x])
    out = {"events": len(x), "unit": "evals/s"}
    k = [0]

    def one(workers):
        p = ((5.0, 0.5, 3.0), (4.9, 0.55, 2.8))[k[0] % 2]
        k[0] += 1
        mean.set(p[0]); sigma.set(p[1]); tau.set(p[2])
        return ref.nll(model, store, ["x0"], workers=workers)

    for workers in (1, cores):
        out[f"workers_{workers}"] = 1.0 / _best_of(lambda w=workers: one(w), reps)
    return out


def run_reference(args) -> None:
    """The reference arm: the reference algorithm's CPU implementation (the
    bit-exact C port, all host threads) on the SAME workload as our arm --
    1e8 events per GPU of our arm generated + weight sum/mean/variance per
    step -- in slices of 2.5e7 rows (global rows, so the events and weights
    are those of one call over the whole step) to bound host memory."""
    import numpy as np

    from oracle import oracle as O  # reference arm (bench infrastructure only)

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    n, sl = EVENTS_PER_GPU * args.gpus, 25_000_000    # our arm's whole-job step: 1e8 events per GPU

    def step():
        s = s2 = 0.0
        for b in range(0, n, sl):
            w = O.generate(DAUGHTERS, M_B0, sl, 1, 1, ev_begin=b, threads=cores)["weight"]
            s += float(np.sum(w))
            s2 += float(np.sum(w * w))
        return s, s2

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s, s2 = step()
    per = (time.perf_counter() - t0) / args.steps
    value = n / per
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(EVENTS_PER_GPU, n),
        "result": {"weight_sum": s, "weight_mean": s / n, "weight_variance": max(s2 / n - (s / n) ** 2, 0.0)},
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": cores, "kind": "port",
                         "sample": f"the full {n:.0e}-event step (2.5e7-row slices), C oracle port, "
                                   f"{cores} pthreads, mean of {args.steps} steps"},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def fcn_bench(hk, torch, evals: int = 200, rank: int = 0, world: int = 1, dist=None) -> dict:
    """FCN evals/s on the 1e7-event gauss+exp data set (configs[3]).  At N
    GPUs the data set is split by row range once and stays resident; every
    eval runs the fused pass over each rank's rows and folds the N partial
    log-sums in rank order (parallel.sharded_nll: one 3-double all-gather),
    so every rank gets the same value.  Strong scaling: total events fixed."""
    from paper_1711_05683_b200 import _lib
    from paper_1711_05683_b200.fitting import lower_model
    from paper_1711_05683_b200.parallel import shard_rows, sharded_nll

    region = hk.BoundedRegion(((0.0, 10.0),))
    mean, sigma, tau = hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5, lower=1e-4), hk.Parameter("tau", 3.0, lower=1e-4)
    g, e = hk.shape_gaussian(mean, sigma), hk.shape_exponential(tau)
    n_sig, n_bkg = hk.Parameter("n_sig", 4e6, lower=0.0), hk.Parameter("n_bkg", 6e6, lower=0.0)
    model = hk.add_pdfs([n_sig, n_bkg], [hk.make_pdf(g, hk.gaussian_norm(g), region),
                                         hk.make_pdf(e, hk.exponential_norm(e), region)])
    data = hk.generate_model_sample(model, hk.RngKey(7, 2), poisson=False)   # exactly 1e7 events, on device
    assert len(data) == FCN_EVENTS
    shard, row0 = shard_rows(data, rank, world)
    n_local = len(shard)
    points = [(5.0, 0.5, 3.0), (4.9, 0.55, 2.8)]

    def one(i):
        p = points[i % 2]
        mean.set(p[0]); sigma.set(p[1]); tau.set(p[2])     # forces host norm recomputation
        return sharded_nll(model, shard, ["x0"], row0)

    for i in range(5):
        one(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(st)
    for i in range(evals):
        one(i)          # returns a host float: the eval is synchronous, as in a minimiser
    ev1.record(st)
    ev1.synchronize()
    dt = ev0.elapsed_time(ev1) * 1e-3 / evals

    def max_over_ranks(v: float) -> float:
        return _max_over_ranks(torch, dist, v)

    dt = max_over_ranks(dt)
    # device-only time of the FCN pass over this rank's rows
    # (the API's kernel -- k_nll_fused, last-CTA fold included -- enqueued back
    # to back without the host wait: hk_nll_eval with no host result)
    x = shard.device_column("x0")
    lm = lower_model(model, x)
    work = torch.zeros(int(_lib.lib().hk_nll_work_doubles(n_local)), dtype=torch.float64, device=x.device)
    for _ in range(3):
        _lib.lib().hk_nll_eval(_lib.ptr(x), n_local, lm, _lib.ptr(work), None, None, st.cuda_stream)
    ev0.record(st)
    for _ in range(evals):
        _lib.lib().hk_nll_eval(_lib.ptr(x), n_local, lm, _lib.ptr(work), None, None, st.cuda_stream)
    ev1.record(st)
    ev1.synchronize()
    kt = max_over_ranks(ev0.elapsed_time(ev1) / evals * 1e-3)
    # the same launch with L2 flushed before each one (a 256 MiB write): the
    # cold-cache kernel, every byte of the column from DRAM
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=x.device)
    cold = []
    for _ in range(20):
        flush.fill_(1.0)
        ev0.record(st)
        _lib.lib().hk_nll_eval(_lib.ptr(x), n_local, lm, _lib.ptr(work), None, None, st.cuda_stream)
        ev1.record(st)
        ev1.synchronize()
        cold.append(ev0.elapsed_time(ev1) * 1e-3)
    kt_cold = max_over_ranks(statistics.median(cold))
    del flush
    # the one-launch C-ABI FCN call alone (kernel + mapped-memory result), no Python
    logsum, first = ctypes.c_double(), ctypes.c_uint64()
    for _ in range(3):
        _lib.lib().hk_nll_eval(_lib.ptr(x), n_local, lm, _lib.ptr(work), ctypes.byref(logsum),
                               ctypes.byref(first), st.cuda_stream)
    c0 = time.perf_counter()
    for _ in range(evals):
        _lib.lib().hk_nll_eval(_lib.ptr(x), n_local, lm, _lib.ptr(work), ctypes.byref(logsum),
                               ctypes.byref(first), st.cuda_stream)
    ct = max_over_ranks((time.perf_counter() - c0) / evals)
    out = {"metric": "FCN evals/s @1e7 events (gauss+exp extended NLL, fp64)", "value": 1.0 / dt,
           "unit": "evals/s", "n_gpus": world, "scaling": "strong", "us_per_eval": dt * 1e6,
           "kernel_us": kt * 1e6, "kernel_us_l2_flushed": kt_cold * 1e6, "c_abi_us": ct * 1e6,
           "l2": "80 MB column < L2; back-to-back calls on the same data as in a fit (no flush)"}
    # the binding roofline: the larger of the two lower bounds on the kernel's
    # time -- HBM (8 B read per event, the observable column) and the FP64
    # pipe (DP instructions per event, ncu) -- with the other as a view
    peak = _peaks()
    hbm = {"bound": "hbm", "achieved": 8 * n_local / kt / 1e9, "peak": peak["hbm_gbs"], "unit": "GB/s",
           "frac": 8 * n_local / kt / 1e9 / peak["hbm_gbs"], "algorithmic_bytes_per_event": 8}
    fp = _fp64_roofline("k_nll_fused", n_local / kt)
    if fp and fp["frac"] > hbm["frac"]:
        out["roofline"] = dict(fp, hbm_view=hbm)
    else:
        out["roofline"] = dict(hbm, **({"fp64_view": fp} if fp else {}))
    if world == 1:
        out.update(fcn_minimiser_paths(hk, torch, model, data, points, (mean, sigma, tau), evals))
    return out


def fcn_minimiser_paths(hk, torch, model, data, points, pars, evals: int) -> dict:
    """The two FCN paths a fit uses besides plain nll(): the resident FCN
    session that fit() opens around the simplex (serial calls, no launch per
    call) and the batched multi-point pass (nll_many: numeric_errors' 51
    Hessian points in one data pass); plus the whole C4 fit's wall time from
    a displaced start (simplex + yield polish + errors)."""
    from paper_1711_05683_b200.fitting import nll_many

    mean, sigma, tau = pars
    res = {}
    with hk.fcn_session(model, data, ["x0"]):
        def one(i):
            p = points[i % 2]
            mean.set(p[0]); sigma.set(p[1]); tau.set(p[2])
            return hk.nll(model, data, ["x0"])
        for i in range(10):
            one(i)
        t0 = time.perf_counter()
        for i in range(evals):
            one(i)
        res["session_evals_per_s"] = evals / (time.perf_counter() - t0)
    ps = model.param_set()
    base = ps.values()
    import numpy as np
    rs = np.random.default_rng(1)
    pts = [tuple(np.asarray(base) * (1 + 1e-4 * rs.standard_normal(len(base)))) for _ in range(51)]
    nll_many(model, data, ["x0"], pts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        nll_many(model, data, ["x0"], pts)
    res["batched51_evals_per_s"] = 51 * 10 / (time.perf_counter() - t0)
    # the batched kernel's FP64 roofline at the API rate (host clock: launch,
    # fold and result read included); the 51 points run as 26 pairs (52)
    rf = _fp64_roofline("k_nll_many", res["batched51_evals_per_s"] / 51 * 52 * len(data))
    if rf:   # frac at the API rate; frac_ncu_one_launch: the kernel alone (52 points)
        res["batched51_fp64"] = {k: rf[k] for k in ("frac", "frac_ncu_one_launch", "dp_inst_per_event")}
    saved = ps.values()
    ps["mean"].set(4.8); ps["sigma"].set(0.6); ps["tau"].set(2.6)
    t0 = time.perf_counter()
    fr = hk.fit(model, data, ["x0"])
    res["fit_s"] = time.perf_counter() - t0
    res["fit_calls"] = fr.n_calls
    res["fit_status"] = fr.status.value
    ps.set_values(saved)
    return res


def write_only_peak(torch) -> float:
    """HBM write-only bandwidth measured live on this GPU: torch fill_ of a
    4 GiB fp64 buffer (>> L2), best of 10, CUDA events -- the north_star's
    "HBM-write roofline" denominator beside MEASURED_PEAKS.json's copy BW."""
    buf = torch.empty(1 << 29, dtype=torch.float64, device="cuda")
    for _ in range(3):
        buf.fill_(1.0)
    best = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(10):
        e0.record()
        buf.fill_(float(i))
        e1.record()
        e1.synchronize()
        best = max(best, buf.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del buf
    torch.cuda.empty_cache()
    return best


def _timed(torch, fn, reps: int, dist=None) -> float:
    """Seconds per call: CUDA events on the current stream, max over ranks."""
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    e1.synchronize()
    return _max_over_ranks(torch, dist, e0.elapsed_time(e1) * 1e-3 / reps)


def _max_over_ranks(torch, dist, v: float) -> float:
    """Max of a per-rank time over the process group (NCCL on device tensors;
    a CPU tensor under the gloo test backend)."""
    if not dist:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def other_configs(hk, torch, _lib, rank: int, world: int, dist) -> dict:
    """The other BASELINE.json configs, measured the same way (secondary
    records, values in events/s unless stated; device-timed with CUDA events,
    max over ranks):
      C1          1e5 events per GPU through phsp_generate (launch + fold bound)
      C2_philox   the C2 generator launch on the Philox4x32-10 production stream
      C3          fused generate + J/psi -> mu mu chain, 1.25e8 events per GPU
                  (1e9 / 8), 17 columns = 136 B/event; frac_copy vs copy BW
      C2_average  phsp_average(<m12^2>) over a stored 1e8 block, 72 B/event read
      CSV         write_csv of 1e7 13-column rows (%.17g formatted on the GPU),
                  rows/s, host wall clock (the text leaves the GPU)
      C5          1e10 events, fused generation + <m12^2>, strong scaling, no
                  event store; 1024 super-chunk records cross GPUs
      C5_bw       the same with <BW_K*(892)(m^2_K pi)> (M=0.89555, G=0.0473)
      C5_generic  1e9 events of <m12^2 * BW(m12^2)>: the NVRTC-specialised
                  kernel, the functor interpreter beside it
      C4_generic  (1 GPU) FCN evals/s at 1e7 events for a Breit-Wigner +
                  polynomial model of closures (the density-program path)
      UNWEIGHT    phsp_unweight of the stored 1e8 block (accept flags + compaction)
      TOYS        (1 GPU) generate_model_sample of the C4 model, 1e7 events
      SPLOT       (1 GPU) ratio_sums and splot_weights over the C4 data set"""
    from paper_1711_05683_b200.parallel import sharded_integrate

    spec, mother = hk.DecaySpec(M_B0, DAUGHTERS), hk.FourVector.at_rest(M_B0)
    out = {}
    # C1: a small block through the public API (launch + fold bound at this size)
    n1 = 100_000

    def c1():
        blk = hk.phsp_generate(spec, mother, n1, hk.RngKey(1, 1), row_offset=rank * n1)
        return blk.meta["weight_partials"]

    dt = _timed(torch, c1, 50, dist)
    out["C1"] = {"value": world * n1 / dt, "ms": dt * 1e3}
    # C2 on the production stream (Philox4x32-10): the same kernel launch as the
    # headline step, device-timed, 104 B/event written
    peak = _peaks()["hbm_gbs"]
    d = _lib.make_decay(spec, mother, M_B0)
    kp = _lib.make_key(hk.RngKey(1, 1), hk.rng.rng_mode("philox"))
    n2 = EVENTS_PER_GPU
    cols = [_lib.empty(n2) for _ in range(13)]
    colp = _lib.ptr_array(cols)
    wp = _lib.empty(2 * _lib.num_weight_slices(n2))
    st = torch.cuda.current_stream()

    def c2p():
        _lib.check(_lib.lib().hk_phsp_generate(d, kp, rank * n2, n2, colp, _lib.ptr(wp), st.cuda_stream), "philox")

    dt = _timed(torch, c2p, 10, dist)
    out["C2_philox"] = {"value": world * n2 / dt, "ms": dt * 1e3, "GBps": BYTES_PER_EVENT * n2 / dt / 1e9,
                        "frac_copy": BYTES_PER_EVENT * n2 / dt / 1e9 / peak}
    del cols, colp, wp
    torch.cuda.empty_cache()
    # C3: fused generate + J/psi -> mu mu chain, 4-body final state, 136 B/event
    n3 = 125_000_000
    sub = hk.DecaySpec(3.0969, (0.1056583755, 0.1056583755))

    def c3():
        return hk.phsp_generate_chain(spec, mother, n3, hk.RngKey(1, 1), 1, sub, hk.RngKey(2, 1),
                                      row_offset=rank * n3)

    c3()
    torch.cuda.empty_cache()
    dt = _timed(torch, c3, 5, dist)
    out["C3"] = {"value": world * n3 / dt, "ms": dt * 1e3, "GBps": 136 * n3 / dt / 1e9,
                 "frac_copy": 136 * n3 / dt / 1e9 / peak}
    torch.cuda.empty_cache()
    # C5: 1e10 events, generation -> m^2_12 -> moments, no store; shards + NCCL gather + fold

    def m12(cols):
        e = cols["p1_e"] + cols["p2_e"]
        px = cols["p1_px"] + cols["p2_px"]
        py = cols["p1_py"] + cols["p2_py"]
        pz = cols["p1_pz"] + cols["p2_pz"]
        return (e * e - px * px - py * py - pz * pz,)

    # C2-average: phsp_average(<m12^2>) over a stored 1e8 block (interpreter over HBM columns:
    # reads p1, p2 four-momenta + weight = 72 B/event)
    blk = hk.phsp_generate(spec, mother, EVENTS_PER_GPU, hk.RngKey(1, 1), row_offset=rank * EVENTS_PER_GPU)
    res = {}

    def c2avg():
        res["r"] = hk.phsp_average(hk.identity(), blk, m12)

    dt = _timed(torch, c2avg, 10, dist)
    out["C2_average"] = {"value": world * EVENTS_PER_GPU / dt, "ms": dt * 1e3,
                         "frac_copy": 72 * EVENTS_PER_GPU / dt / 1e9 / peak}
    # UNWEIGHT: accept-reject of the stored 1e8 block against
    # phsp_max_weight, order-preserving compaction of the accepted rows
    w_max = hk.phsp_max_weight(spec)
    acc = {}

    def unw():
        acc.pop("b", None)  # free the last result first: no allocator growth in the timed region
        acc["b"] = hk.phsp_unweight(blk, w_max, hk.RngKey(1, 4), row_offset=rank * EVENTS_PER_GPU)

    dt = _timed(torch, unw, 5, dist)
    n_acc = len(acc.pop("b"))
    # flags: 8 B weight read + 1 B flag written; compaction: 1 B flag + 13 columns read
    # and written for each accepted row (flag scan and counts are negligible)
    ub = 9 * EVENTS_PER_GPU + EVENTS_PER_GPU + 2 * 104 * n_acc
    out["UNWEIGHT"] = {"value": world * EVENTS_PER_GPU / dt, "ms": dt * 1e3, "accepted": n_acc,
                       "frac_copy": ub / dt / 1e9 / peak}
    # CSV: write_csv of 1e7 stored rows, GPU-formatted text streamed to a file
    from paper_1711_05683_b200.store import ColumnStore
    n_csv = 10_000_000
    sub = ColumnStore._from_device(blk.schema, [c[:n_csv] for c in blk.device_columns()])
    with open(os.devnull, "wb") as fh:
        sub.write_csv(fh)                     # warm-up (allocations)
        t0 = time.perf_counter()
        sub.write_csv(fh)
        dt = time.perf_counter() - t0
    out["CSV"] = {"value": n_csv / dt, "unit": "rows/s"}
    del sub
    del blk
    torch.cuda.empty_cache()
    n5 = 10_000_000_000
    res = {}

    def c5():
        res["r"] = sharded_integrate(hk.identity(), spec, mother, n5, hk.RngKey(1, 1), m12)

    dt = _timed(torch, c5, 2, dist)
    rf = _fp64_roofline("hk_jit_integrate", n5 / dt / world)
    out["C5"] = {"value": n5 / dt, "s": dt, "fp64_frac": rf["frac"] if rf else None}
    # C5 secondary integrand: K*(892) Breit-Wigner on m^2_K pi, the named builtin

    def m23(cols):
        e = cols["p2_e"] + cols["p3_e"]
        px = cols["p2_px"] + cols["p3_px"]
        py = cols["p2_py"] + cols["p3_py"]
        pz = cols["p2_pz"] + cols["p3_pz"]
        return (e * e - px * px - py * py - pz * pz,)

    def c5bw():
        res["r"] = sharded_integrate(hk.breit_wigner(0.89555, 0.0473), spec, mother, n5, hk.RngKey(1, 1), m23)

    dt = _timed(torch, c5bw, 2, dist)
    out["C5_bw"] = {"value": n5 / dt}
    # C5 with an integrand outside the recognised Dalitz shapes: m12^2 * BW(m12^2)
    # runs as a specialised (NVRTC) kernel; the interpreter is timed beside it.
    expr = hk.identity() * hk.breit_wigner(3.0969, 0.1)
    n5g = 1_000_000_000 // world

    def c5g():
        return hk.phsp_integrate(expr, spec, mother, n5g, hk.RngKey(1, 1), m12, row_offset=rank * n5g,
                                 return_partials=True)

    dt_jit = _timed(torch, c5g, 3, dist)
    with _lib.jit_mode(_lib.JIT_OFF):
        dt_int = _timed(torch, c5g, 1, dist)
    out["C5_generic"] = {"value": world * n5g / dt_jit, "interpreter": world * n5g / dt_int}
    if world == 1:
        out["C4_generic"] = fcn_generic(hk, torch)
        out["TOYS"] = toy_sample(hk, torch)
        out["SPLOT"] = splot_pass(hk, torch)
    return out


def splot_pass(hk, torch) -> dict:
    """SURVEY 8f rank 2 on the C4 data set (1e7 events): the yield-stationarity
    / sWeights-matrix accumulation (ratio_sums: K + K^2 sums per event, 8 B
    read) and the per-event sWeights table (splot_weights: 8 B read, 8 K B
    written), rows/s with CUDA events, HBM fraction of copy BW."""
    import numpy as np

    from paper_1711_05683_b200.fitting import ratio_sums
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(P("mean", 5.0), P("sigma", 0.5))
    e = hk.shape_exponential(P("tau", 3.0))
    model = hk.add_pdfs([P("n_sig", 4e6), P("n_bkg", 6e6)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
    data = hk.generate_model_sample(model, hk.RngKey(7, 2), poisson=False)
    n = len(data)
    peak = _peaks()["hbm_gbs"]
    dt_sums = _timed(torch, lambda: ratio_sums(model, data, ["x0"]), 20)
    V = np.eye(2)
    dt_w = _timed(torch, lambda: hk.splot_weights(model, data, ["x0"], V), 20)
    return {"what": "C4 data set (1e7): ratio_sums (yields / sWeights matrix) and splot_weights",
            "ratio_sums_rows_per_s": n / dt_sums, "splot_weights_rows_per_s": n / dt_w,
            "ratio_sums_frac_copy": 8 * n / dt_sums / 1e9 / peak,
            "splot_weights_frac_copy": 24 * n / dt_w / 1e9 / peak}


def toy_sample(hk, torch) -> dict:
    """the C4 data set itself -- generate_model_sample of
    the benchmark model (build_model(scale=200): 4e6 Gaussian + 6e6
    exponential events, RngKey(7, 2), poisson=False; fitting.py:526-552) by
    device accept-reject, events/s (host wall clock around the API call)."""
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(P("mean", 5.0), P("sigma", 0.5))
    e = hk.shape_exponential(P("tau", 3.0))
    model = hk.add_pdfs([P("n_sig", 4e6), P("n_bkg", 6e6)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
    for _ in range(2):
        data = hk.generate_model_sample(model, hk.RngKey(7, 2), poisson=False)
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        data = hk.generate_model_sample(model, hk.RngKey(7, 2), poisson=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    return {"what": "generate_model_sample of the C4 model, 1e7 events (device accept-reject)",
            "value": len(data) / dt, "ms": dt * 1e3}


def fcn_generic(hk, torch, n: int = FCN_EVENTS, evals: int = 200, keep: bool = False) -> dict:
    """FCN evals/s at 1e7 events for a model outside the closed-form kernels:
    a Breit-Wigner + linear polynomial of wrap_closure shapes (the reference's
    nll accepts any Pdf shape, fitting.py:160-166), lowered once to a
    parametric density program and run as an NVRTC-specialised kernel; the
    parameters change every call (norms recomputed on the host)."""
    import math

    import numpy as np
    P = hk.Parameter
    lo, hi = 0.6, 1.2
    m0, g, c0, c1 = P("m0", 0.8955), P("g", 0.0473), P("c0", 1.0), P("c1", 0.5)
    bw = hk.wrap_closure(lambda x, p: 1.0 / ((x[0] - p["m0"].value) ** 2 + (0.5 * p["g"].value) ** 2), [m0, g])
    poly = hk.wrap_closure(lambda x, p: p["c0"].value + p["c1"].value * x[0], [c0, c1])
    region = hk.BoundedRegion(((lo, hi),))

    def bw_norm(r):
        h = 0.5 * g.value
        return (math.atan((hi - m0.value) / h) - math.atan((lo - m0.value) / h)) / h

    model = hk.add_pdfs([P("n_bw", 0.3 * n), P("n_poly", 0.7 * n)],
                        [hk.make_pdf(bw, bw_norm, region),
                         hk.make_pdf(poly, lambda r: c0.value * (hi - lo) + 0.5 * c1.value * (hi * hi - lo * lo),
                                     region)])
    x = np.random.default_rng(11).uniform(lo, hi, n)
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    points = [(0.8955, 0.0473), (0.8900, 0.0500)]

    def one(i):
        m0.set(points[i % 2][0]); g.set(points[i % 2][1])
        return hk.nll(model, data, ["x0"])

    for i in range(5):
        one(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(evals):
        one(i)
    dt = (time.perf_counter() - t0) / evals
    out = {"what": "FCN @1e7 events, Breit-Wigner + linear polynomial closures (NVRTC density program)",
           "value": 1.0 / dt, "unit": "evals/s", "us_per_eval": dt * 1e6}
    if keep:
        out.update(_model=model, _data=data)
    return out


def run_ours(args) -> None:
    import numpy as np
    import torch

    import paper_1711_05683_b200 as hk
    from paper_1711_05683_b200 import _lib
    from paper_1711_05683_b200.parallel import gather_supers, shard_range, super_span

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HK_BENCH_BACKEND=gloo + HK_BENCH_DEVICE=0: exercise the N>1 code path with
    # several ranks on one GPU (independent kernels, CPU collectives) -- a
    # correctness check of the multi-rank plumbing, never a bench number
    local = int(os.environ.get("HK_BENCH_DEVICE", local))
    backend = os.environ.get("HK_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    spec, mother = hk.DecaySpec(M_B0, DAUGHTERS), hk.FourVector.at_rest(M_B0)
    n_total = EVENTS_PER_GPU * world
    row0, row1 = shard_range(n_total, rank, world)    # whole super-chunks: 1e8 rows per rank up to a chunk
    s0, s1 = super_span(rank, world)
    n = row1 - row0
    key = hk.RngKey(1, 1)
    d = _lib.make_decay(spec, mother, M_B0)
    k = _lib.make_key(key)
    cols = [_lib.empty(n) for _ in range(13)]
    colp = _lib.ptr_array(cols)
    wpart = _lib.empty(2 * _lib.num_weight_slices(n))
    st = torch.cuda.current_stream()
    L = _lib.lib()

    def step(gen_events=None):
        if gen_events:
            gen_events[0].record(st)
        _lib.check(L.hk_phsp_generate(d, k, row0, n, colp, _lib.ptr(wpart), st.cuda_stream), "generate")
        if gen_events:
            gen_events[1].record(st)
        local = _lib.fold_supers(wpart, n_total, s0, s1, _lib.HK_WARP_SLICES, 2)   # warp slices -> supers
        full, _ = gather_supers(local, 2)                  # 1024 x 16 B cross GPUs
        return _lib.fold(full, _lib.HK_SUPERS, 2)

    for _ in range(args.warmup):
        tot = step()
    torch.cuda.synchronize()
    gen_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with NvmlClockSampler(local) as clocks:
        t0.record(st)
        for i in range(args.steps):
            tot = step(gen_ev[i])
        t1.record(st)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed = t0.elapsed_time(t1) * 1e-3
    gen_times = [a.elapsed_time(b) * 1e-3 for a, b in gen_ev]
    elapsed = _max_over_ranks(torch, dist, elapsed)
    sums = tot.cpu().numpy()
    per_step = elapsed / args.steps
    value = n_total / per_step
    gen_avg = sum(gen_times) / len(gen_times)
    peaks = _peaks()
    achieved = BYTES_PER_EVENT * n / gen_avg / 1e9
    traffic = _traffic()

    del cols
    torch.cuda.empty_cache()
    write_peak = None if args.no_peaks else write_only_peak(torch)
    # end to end through the public API, host buffers (pinned), D2H inside the timed region
    e2e = None
    if rank == 0 or world > 1:
        # N > 1: 1e8 / N events per rank, so the job pins ~10.4 GB of host
        # memory in total at any N (the leg is PCIe-bound per GPU; the rate
        # does not depend on the per-rank size)
        n_e = n if world == 1 else max(4096, n // world // 4096 * 4096)
        host = [torch.empty(n_e, dtype=torch.float64, pin_memory=True) for _ in range(13)]
        hk.phsp_generate_to_host(spec, mother, n_e, key, row_offset=rank * n_e, out=host)   # warm (staging alloc)
        e_steps = max(1, min(args.steps, 5))
        torch.cuda.synchronize()
        a0 = time.perf_counter()
        for _ in range(e_steps):
            _, ws = hk.phsp_generate_to_host(spec, mother, n_e, key, row_offset=rank * n_e, out=host)
        e_dt = (time.perf_counter() - a0) / e_steps
        e2e = {"value": world * n_e / e_dt if world == 1 else None, "per_gpu_value": n_e / e_dt,
               "unit": "events/s", "events_per_rank": n_e,
               "h2d_bytes_per_step": ctypes.sizeof(_lib.hk_decay_t) + ctypes.sizeof(_lib.hk_key_t),
               "d2h_bytes_per_step": BYTES_PER_EVENT * n_e + 16,
               "api": "phsp_generate_to_host: pinned host columns, D2H overlapped with generation",
               "steps": e_steps}
        if dist:
            e2e["value"] = world * n_e / _max_over_ranks(torch, dist, e_dt)
        # the ceiling this leg runs into: raw device->host copy into pinned memory
        raw = host[0].view(torch.uint8)
        dev_src = torch.empty(raw.numel(), dtype=torch.uint8, device="cuda")
        raw.copy_(dev_src)
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        for _ in range(3):
            raw.copy_(dev_src, non_blocking=True)
        torch.cuda.synchronize()
        ceiling = 3 * raw.numel() / (time.perf_counter() - c0) / 1e9
        e2e["d2h_ceiling_GBps"] = ceiling
        e2e["d2h_GBps"] = (BYTES_PER_EVENT * n_e + 16) / e_dt / 1e9
        e2e["frac_of_d2h_ceiling"] = e2e["d2h_GBps"] / ceiling
        del dev_src, raw
        del host
        torch.cuda.empty_cache()
        # the drop-in API as a user calls it: phsp_generate (device-resident
        # store) + phsp_weight_moments (the step's result, 16 B read back)
        def api_step():
            blk = hk.phsp_generate(spec, mother, n, key, row_offset=row0)
            return hk.phsp_weight_moments(blk)

        api_step()
        torch.cuda.synchronize()
        a0 = time.perf_counter()
        for _ in range(e_steps):
            api_step()
        a_dt = _max_over_ranks(torch, dist, (time.perf_counter() - a0) / e_steps)
        e2e["api_device_resident"] = {
            "value": n_total / a_dt, "unit": "events/s",
            "api": "phsp_generate -> phsp_weight_moments, events stay in HBM",
            "d2h_bytes_per_step": 16}

    others = None if args.no_configs else other_configs(hk, torch, _lib, rank, world, dist)
    fcn = None if args.no_fcn else fcn_bench(hk, torch, evals=args.fcn_evals, rank=rank, world=world, dist=dist)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(n, n_total),
            "parallelism": f"dp{world}: contiguous super-chunk-aligned event shards, NCCL all-gather of 1024 super-chunk records",
            "result": {"weight_sum": float(sums[0]), "weight_mean": float(sums[0] / n_total),
                       "weight_variance": float(max(sums[1] / n_total - (sums[0] / n_total) ** 2, 0.0))},
            "roofline": {"bound": "hbm", "kernel": "k_generate<3, reference>", "achieved": achieved,
                         "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                         "peak_source": peaks["source"], "traffic": traffic,
                         "algorithmic_bytes_per_event": BYTES_PER_EVENT,
                         "kernel_ms": gen_avg * 1e3, "kernel_share_of_step": gen_avg / per_step,
                         "write_only_peak": write_peak,
                         "frac_vs_write_only": achieved / write_peak if write_peak else None},
            "clocks": clocks.summary(),
            "e2e": e2e,
            "gpu_launches": 3 * args.steps,   # k_generate + k_fold_supers + k_fold per step
            "cpu_baseline": cpu,
            "other_configs": others,
            "fcn": fcn,      # last: the driver keeps the tail of the line
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-fcn", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--fcn-evals", type=int, default=200)
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C3/C5 secondary measurements")
    ap.add_argument("--no-peaks", action="store_true",
                    help="skip the live write-only HBM measurement (its fill kernels would join an ncu launch list)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

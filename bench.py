#!/usr/bin/env python
"""Benchmark of the filtered PIM matrix exponential (arXiv 2110.04493) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 5] [--plan-norm one|fro] [--eps-tol 1e-16]

One step = one whole e^H through the C ABI: sexpm_plan (validation, device norm,
Eq. 4.20 plan, H0 = H 2^-N) + sexpm_run (filtered Taylor phase, N filtered squarings,
E = I + T^_N) + sexpm_destroy, with H resident in HBM.  Workload: BASELINE.json config 5
(n = 1449^2 2D Dirichlet heat, r = 0.5, the configuration the north-star target names),
synthetic and seeded.  N > 1: torchrun, one rank per GPU, contiguous row blocks with an
NCCL halo exchange per squaring (strong scaling: the job is one e^H).

Prints ONE JSON line on rank 0.  `value` = e^H per second for the whole job (K / max over
ranks of the device time of the K timed steps).  See DESIGN.md "Measurement".
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

METRIC = "e^H wall time & squarings/s; achieved HBM GB/s vs peak, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--plan-norm", default="one", choices=["one", "fro"])
    ap.add_argument("--eps-tol", type=float, default=1e-16)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-apply", action="store_true", help="skip the N1 apply measurement")
    ap.add_argument("--no-n2", action="store_true", help="skip the N2 filter-off comparison")
    ap.add_argument("--no-n3", action="store_true", help="skip the N3 reordering comparison")
    ap.add_argument("--no-n4", action="store_true", help="skip the N4 graph workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-others", action="store_true", help="skip configs 2-4 and the F-norm plan")
    ap.add_argument("--cpu-sample-grid", type=int, default=0)
    return ap.parse_args()


# ---------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        import statistics
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------------------
CPU_SAMPLE_GRID = {5: 256, 2: 100, 1: 1000, 3: 100, 4: 20}


def sample_config(args):
    """The bounded sample of the workload both the CPU baseline and the reference arm time:
    the same law as the benched config on a smaller grid (config 5: the uniform 2D Dirichlet
    heat matrix r = 0.5 on a 256 x 256 grid, n = 65536), same eps_tol and plan norm."""
    from synth import make_config
    g = args.cpu_sample_grid or CPU_SAMPLE_GRID.get(args.config, 64)
    return make_config(args.config, scale_down=g), g


def cpu_oracle_sample(args, H=None, g=None):
    """One e^H of the sample by the oracle as it stands (OpenMP over rows, all host cores):
    (e^H/s of the sample as measured, cores, description, seconds).  Not scaled."""
    import oracle as O
    if H is None:
        H, g = sample_config(args)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    O.expm(H, args.eps_tol, plan_norm=args.plan_norm, nthreads=cores)
    dt = time.perf_counter() - t0
    desc = (f"one e^H of the config-{args.config} law on a {g}x{g} grid (n={H.n}, eps_tol "
            f"{args.eps_tol:g}, {args.plan_norm}-norm plan), oracle with {cores} OpenMP threads; "
            "measured, not scaled")
    return 1.0 / dt, cores, desc, dt


def make_config_n(cid):
    from synth.configs import CONFIGS
    return CONFIGS[cid]["n"]


def run_reference(args):
    """The reference arm for this tier: the CPU oracle (oracle/, as it stands) on the box's
    host cores; each step = one e^H of the bounded sample of the workload (sample_config),
    timed whole; value = e^H/s of that sample (our line reports the GPU on the same sample
    under "same_sample")."""
    rank, world, _ = dist_env()
    if rank != 0:
        return  # other ranks exit without work
    H, g = sample_config(args)
    times = []
    for i in range(args.warmup + args.steps):
        v, cores, sample, dt = cpu_oracle_sample(args, H, g)
        if i >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = 1000.0 / ms
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "e^H/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"BASELINE config {args.config} law on a {g}x{g} grid (n={H.n}): "
                                   "the bounded CPU sample of the benched workload",
                       "eps_tol": args.eps_tol, "plan_norm": args.plan_norm},
            "cpu_baseline": {"value": value, "unit": "e^H/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "e^H/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2110_04493_b200 import binding as B
    from paper_2110_04493_b200.build import build
    if rank == 0:
        build()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    B.lib()
    # fp64 roofline denominators measured on this GPU (DFMA chains and DMMA accumulators)
    fp64_peak = B.sexpm_fp64_peak()
    FP64_PEAK_TFLOPS = fp64_peak["dfma_tflops"]
    from synth import make_config
    H = make_config(args.config)
    n = H.n
    comm = None
    if world > 1:
        import torch.distributed as dist
        uid = [B.sexpm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = B.sexpm_nccl_comm_init(rank, world, uid[0])
        # contiguous row blocks balanced by a squaring-work proxy (row nnz^2)
        w = np.diff(H.rowptr).astype(np.float64) ** 2
        bounds = B.sexpm_partition_rows(n, w, world)
    else:
        bounds = np.array([0, n], np.int64)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    Hl = H.rows(r0, r1)
    rp = torch.from_numpy(Hl.rowptr).to(dev)
    ci = torch.from_numpy(Hl.col).to(dev)
    va = torch.from_numpy(Hl.val).to(dev)
    stream = torch.cuda.current_stream()
    opts = dict(plan_norm=args.plan_norm)
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def one_step():
        p = B.Plan(n, rp, ci, va, args.eps_tol, row_begin=r0, row_end=r1, nccl_comm=comm,
                   stream=stream, **opts)
        out = p.run_only()
        st = p.stats()
        p.close()
        return out, st

    for _ in range(args.warmup):
        one_step()
    barrier()
    launches0 = B.sexpm_kernel_launches()
    times = []
    stats = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            l2_flush.zero_()  # flush L2 between timed steps (outside the timed span)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out, st = one_step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            stats.append(st)
        barrier()
    launches = B.sexpm_kernel_launches() - launches0
    total_ms = sum(times)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = 1000.0 / ms_per_step
    st = stats[-1]
    N = int(st["N"])

    # ---------------- end to end through the C ABI with HOST buffers ----------------
    e2e = None
    est_out_bytes = int(st["nnz_out"]) * 12 + (r1 - r0 + 1) * 8
    try:
        avail = int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0].split()[1]) * 1024
    except Exception:
        avail = 0
    if est_out_bytes > 0.25 * avail:
        e2e = {"value": None, "unit": "e^H/s", "skipped": f"pinned result buffer {est_out_bytes/1e9:.1f} GB > 25% of host MemAvailable {avail/1e9:.1f} GB"}
    elif not args.no_e2e:
        hrp = torch.from_numpy(Hl.rowptr).pin_memory().numpy()
        hci = torch.from_numpy(Hl.col).pin_memory().numpy()
        hva = torch.from_numpy(Hl.val).pin_memory().numpy()
        nnz_out = int(st["nnz_out"]) if world == 1 else None
        outbufs = None
        e2e_times = []
        h2d = hrp.nbytes + hci.nbytes + hva.nbytes
        d2h = 0
        for it in range(2 if world == 1 else 0):
            barrier()
            t0 = time.perf_counter()
            o = B.sexpm_options_init(plan_norm=args.plan_norm)
            o.stream = B.stream_handle(stream)
            Hin = B._csr_in(n, hrp, hci, hva, r0, r1, host=True)
            h = B.sexpm_plan_host(Hin, args.eps_tol, o)
            E = B.sexpm_run(h)
            if outbufs is None or outbufs[1].numel() < E.nnz:
                if it > 0:  # never copy into a buffer that is too small
                    e2e_times = []
                cap = int(E.nnz * 1.01) + 1024
                outbufs = (torch.empty(r1 - r0 + 1, dtype=torch.int64).pin_memory(),
                           torch.empty(cap, dtype=torch.int32).pin_memory(),
                           torch.empty(cap, dtype=torch.float64).pin_memory())
                if it == 0:
                    B.sexpm_destroy(h)
                    continue  # first pass only sizes the pinned buffers
            B.sexpm_result_copy(h, outbufs[0].data_ptr(), outbufs[1].data_ptr(), outbufs[2].data_ptr())
            B.sexpm_destroy(h)
            torch.cuda.synchronize()
            e2e_times.append(time.perf_counter() - t0)
            d2h = (r1 - r0 + 1) * 8 + E.nnz * 12
        if e2e_times:
            serial = 1.0 / min(e2e_times)
            e2e = {"value": serial, "unit": "e^H/s", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h),
                   "note": "sexpm_plan_host (H2D of H from pinned memory) + sexpm_run + "
                           "sexpm_result_copy (D2H of E into pinned memory), wall clock"}
            # Consecutive e^H through sexpm_result_copy_async: step k's D2H of E (copy stream,
            # its own pinned buffer set) overlaps step k+1's H2D + plan + run.  Every step's
            # H2D and D2H lie inside the timed region, which ends when the last copy has
            # landed.  The one-shot figure above stays as `serial_value`.
            if 2 * est_out_bytes <= 0.5 * avail:
                ke, kw = max(8, min(args.steps, 16)), 3

                def pipelined(k, mark_at):
                    """k consecutive e^H; returns the wall time from the start of step mark_at
                    (whose predecessor's copy is then in flight) until the last copy has landed."""
                    pending = None
                    t_mark = None
                    for i in range(k):
                        if i == mark_at:
                            t_mark = time.perf_counter()
                        o = B.sexpm_options_init(plan_norm=args.plan_norm)
                        o.stream = B.stream_handle(stream)
                        Hin = B._csr_in(n, hrp, hci, hva, r0, r1, host=True)
                        h = B.sexpm_plan_host(Hin, args.eps_tol, o)
                        E = B.sexpm_run(h)
                        assert E.nnz <= sets[0][1].numel()
                        if pending is not None:
                            B.sexpm_result_wait(pending)
                        bs = sets[i % 2]
                        pending = B.sexpm_result_copy_async(h, bs[0].data_ptr(), bs[1].data_ptr(),
                                                            bs[2].data_ptr())
                        B.sexpm_destroy(h)
                    B.sexpm_result_wait(pending)
                    torch.cuda.synchronize()
                    return time.perf_counter() - t_mark

                # kw untimed steps first (the second result's device blocks enter the cache), then
                # ke timed steps of the same pipeline, the drain of the last copy included
                barrier()
                sets = None
                try:
                    sets = [outbufs, tuple(torch.empty_like(t).pin_memory() for t in outbufs)]
                    dt = pipelined(kw + ke, kw)
                except Exception as ex:  # keep the one-shot figure; say why the pipeline did not run
                    dt = None
                    e2e["pipelined_error"] = f"{type(ex).__name__}: {ex}"[:300]
                    try:
                        torch.cuda.synchronize()
                        B.sexpm_release_cache()
                    except Exception:
                        pass
                nz = int(st["nnz_out"])
                same = dt is not None and (torch.equal(sets[0][0], sets[1][0]) and torch.equal(sets[0][1][:nz], sets[1][1][:nz])
                        and torch.equal(sets[0][2][:nz], sets[1][2][:nz]))
                if dt is not None:
                  e2e.update({"value": ke / dt, "serial_value": serial, "pipelined_steps": ke,
                            "pipelined_identical_results": bool(same),
                            "pipelined_warmup_steps": kw,
                            "note": f"{ke} consecutive e^H (after {kw} untimed ones of the same "
                                    "pipeline), each sexpm_plan_host (H2D of H from pinned "
                                    "memory) + sexpm_run + sexpm_result_copy_async (D2H of E into one "
                                    "of two pinned buffer sets by k_copy_out, overlapping the next "
                                    "e^H) + sexpm_destroy; wall clock from the first timed step's "
                                    f"start until the last copy has landed, / {ke}.  serial_value: "
                                    "one e^H with the blocking sexpm_result_copy"})

    # ---------------- N1 apply: Y = E X on the device ----------------
    # one e^H, then Y = E X for a seeded dense X of m columns; CUDA events around each call
    # (E = 14.6 GB >> L2, L2 flushed anyway); compulsory bytes = E + rowptr + X + Y
    apply_res = None
    peaks0 = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    if world == 1 and not args.no_apply:
        p = B.Plan(n, rp, ci, va, args.eps_tol, stream=stream, **opts)
        p.run_only()
        nnzE = int(p.stats()["nnz_out"])
        gen = torch.Generator(device=dev)
        gen.manual_seed(20211010)
        apply_res = {"kernel": "k_spmm (warp per row, lanes over columns)", "nnz_E": nnzE}
        for m in (1, 64):
            X = torch.randn((n, m), dtype=torch.float64, device=dev, generator=gen)
            Y = torch.empty_like(X)
            p.apply(X, Y=Y)
            ts = []
            for _ in range(5):
                l2_flush.zero_()
                torch.cuda.synchronize()
                a0 = torch.cuda.Event(enable_timing=True)
                a1 = torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                p.apply(X, Y=Y)
                a1.record(stream)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(a1))
            ms = sorted(ts)[len(ts) // 2]
            byts = 12.0 * nnzE + 8.0 * (n + 1) + 16.0 * n * m
            fl = 2.0 * nnzE * m
            hp = peaks0.get("hbm_gbs", 6650.0)
            apply_res[f"m{m}"] = {"ms": ms, "hbm_gbs_compulsory": byts / ms / 1e6,
                                  "hbm_frac": byts / ms / 1e6 / hp,
                                  "fp64_tflops": fl / ms / 1e9, "fp64_frac": fl / ms / 1e9 / FP64_PEAK_TFLOPS}
            del X, Y
        p.close()

    # ---------------- N2: what the filter saves ----------------
    # BASELINE config 2 (n = 10^4) with the paper's filter and with it off (the unfiltered
    # PIM: every eps_g = 0): nnz per squaring, device time; config 5 unfiltered would need
    # ~10^4 entries per row (bandwidth doubling per squaring, Table 3's unfiltered row).
    n2 = None
    if world == 1 and not args.no_n2:
        H2 = make_config(2)
        r2 = [torch.from_numpy(a).to(dev) for a in (H2.rowptr, H2.col, H2.val)]
        n2 = {"workload": "BASELINE config 2 (2D heat 100x100, perturbed), eps_tol 1e-16"}
        for name, flt in (("filtered", 1), ("unfiltered", 0)):
            ts = []
            reps = 3 if flt else 1  # the unfiltered run takes seconds: one pass
            for rep_i in range(reps):
                p = B.Plan(H2.n, *r2, args.eps_tol, stream=stream, filter=flt, **opts)
                b0 = torch.cuda.Event(enable_timing=True)
                b1 = torch.cuda.Event(enable_timing=True)
                b0.record(stream)
                p.run_only()
                b1.record(stream)
                torch.cuda.synchronize()
                s2 = p.stats()
                p.close()
                if rep_i or reps == 1:
                    ts.append(b0.elapsed_time(b1))
            N2 = int(s2["N"])
            n2[name] = {"ms": min(ts), "nnz_E": int(s2["nnz_out"]),
                        "sq_nnz": [int(x) for x in s2["sq_nnz"][0:N2 + 1]],
                        "sq_bandwidth_l1": [int(x) for x in s2["sq_l1"][0:N2 + 1]],
                        "sq_fmas": float(sum(s2["sq_fmas"][1:N2 + 1]))}

    # ---------------- N3: reordering a scrambled input ----------------
    # BASELINE config 3 (structural, n = 1.8e5) under a seeded random relabelling: e^H as
    # given and with option reorder (device RCM, run on P H P^T, E mapped back)
    n3 = None
    if world == 1 and not args.no_n3:
        import scipy.sparse as sps
        H3 = make_config(3)
        q = np.random.default_rng(20211010).permutation(H3.n)
        A3 = sps.csr_matrix((H3.val, H3.col, H3.rowptr), shape=(H3.n, H3.n))[q][:, q].tocsr()
        A3.sort_indices()
        r3 = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in
              (A3.indptr.astype(np.int64), A3.indices.astype(np.int32), A3.data.astype(np.float64))]
        n3 = {"workload": "BASELINE config 3 (structural 300x300, n = 180000) under a random relabelling"}
        for name, ro in (("as_given", 0), ("reorder_rcm", 1)):
            ts, tp = [], []
            for rep_i in range(2):
                b0 = torch.cuda.Event(enable_timing=True)
                b1 = torch.cuda.Event(enable_timing=True)
                b2 = torch.cuda.Event(enable_timing=True)
                b0.record(stream)
                p = B.Plan(H3.n, *r3, args.eps_tol, stream=stream, reorder=ro, **opts)
                b1.record(stream)
                p.run_only()
                b2.record(stream)
                torch.cuda.synchronize()
                s3 = p.stats()
                p.close()
                if rep_i:
                    ts.append(b0.elapsed_time(b2))
                    tp.append(b0.elapsed_time(b1))
            N3 = int(s3["N"])
            n3[name] = {"ms_plan_plus_run": min(ts), "ms_plan": min(tp), "nnz_E": int(s3["nnz_out"]),
                        "bandwidth_l1_T0": int(s3["sq_l1"][0]),
                        "sq_fallback_rows": [int(x) for x in s3["sq_fallback_rows"][1:N3 + 1]]}

    # ---------------- N4: an unstructured graph workload ----------------
    # communicability e^{beta A} of a random geometric graph (n = 2e5, mean degree 6,
    # ||H||_1 = 4, random node order), with the device RCM (option reorder) and as given
    n4 = None
    if world == 1 and not args.no_n4:
        from synth import geometric_graph
        G4 = geometric_graph(200000, 6.0, 4.0, 20211010)
        r4 = [torch.from_numpy(a).to(dev) for a in (G4.rowptr, G4.col, G4.val)]
        n4 = {"workload": "random geometric graph n=200000, mean degree 6, H = beta A, ||H||_1 = 4, random node order",
              "nnz_H": int(G4.nnz)}
        for name, ro in (("reorder_rcm", 1), ("as_given", 0)):
            ts = []
            for rep_i in range(2 if ro else 1):
                b0 = torch.cuda.Event(enable_timing=True)
                b1 = torch.cuda.Event(enable_timing=True)
                b0.record(stream)
                p = B.Plan(G4.n, *r4, args.eps_tol, stream=stream, reorder=ro, **opts)
                p.run_only()
                b1.record(stream)
                torch.cuda.synchronize()
                s4 = p.stats()
                p.close()
                if rep_i or not ro:
                    ts.append(b0.elapsed_time(b1))
                    ph = {"plan": float(s4["ms_plan"]), "taylor": float(s4["ms_taylor"]),
                          "squaring": float(s4["ms_squaring"])}
            N4 = int(s4["N"])
            n4[name] = {"ms_plan_plus_run": min(ts), "phase_ms": ph, "M": int(s4["M"]), "N": N4,
                        "nnz_E": int(s4["nnz_out"]),
                        "bandwidth_l1_T0": int(s4["sq_l1"][0]),
                        "sq_fallback_rows": [int(x) for x in s4["sq_fallback_rows"][1:N4 + 1]]}

    # ---------------- the other configurations (one GPU; outside the timed steps) --------
    # e^H (plan + run) device time of BASELINE configs 2-4 and of config 5 with the paper's
    # Frobenius-norm plan ((M, N) = (19, 12)), best of 2 after a warm-up run
    others = None
    if world == 1 and not args.no_others:
        others = {}
        cases = [("config5_fro_plan", 5, "fro"), ("config2", 2, "one"), ("config3", 3, "one"),
                 ("config4", 4, "one")]
        for name, cid, pn in cases:
            if cid == args.config and pn == args.plan_norm:
                continue
            Hc = H if cid == args.config else make_config(cid)
            rc = [torch.from_numpy(a).to(dev) for a in (Hc.rowptr, Hc.col, Hc.val)]
            ts = []
            for rep_i in range(3):
                b0 = torch.cuda.Event(enable_timing=True)
                b1 = torch.cuda.Event(enable_timing=True)
                b0.record(stream)
                p = B.Plan(Hc.n, *rc, args.eps_tol, stream=stream, plan_norm=pn)
                p.run_only()
                b1.record(stream)
                torch.cuda.synchronize()
                sc = p.stats()
                p.close()
                if rep_i:
                    ts.append(b0.elapsed_time(b1))
            Nc = int(sc["N"])
            sqk = [float(x) for x in sc["sq_kernel_ms"][1:Nc + 1]]
            sqf = [2.0 * float(x) for x in sc["sq_fmas"][1:Nc + 1]]
            others[name] = {"n": Hc.n, "plan_norm": pn, "M": int(sc["M"]), "N": Nc,
                            "ms_expm": min(ts), "e_per_s": 1000.0 / min(ts),
                            "phase_ms": {"plan": float(sc["ms_plan"]), "taylor": float(sc["ms_taylor"]),
                                         "squaring": float(sc["ms_squaring"]), "finalize": float(sc["ms_finalize"])},
                            "squarings_per_s": Nc / (float(sum(sc["sq_ms"][1:Nc + 1])) / 1e3) if Nc else None,
                            "sq_kernel_ms": sqk,
                            "sq_fp64_tflops_algorithmic": [f / (m * 1e9) for f, m in zip(sqf, sqk) if m > 0],
                            "sq_fallback_rows": [int(x) for x in sc["sq_fallback_rows"][1:Nc + 1]],
                            "nnz_E": int(sc["nnz_out"])}
            del rc

    # ---------------- config S (HBM-roofline case, 1D rows) ----------------
    # 0.5 tridiag(1,-2,1) at n = 2^25 (2^26 exceeds the device memory with the staging pool
    # and the padded Taylor accumulator), built on the device; one warm-up, one timed run
    config_s = None
    if world == 1 and not args.no_others:
        ns = 1 << 25
        r_ = torch.arange(ns, device=dev, dtype=torch.int64)
        cnt_ = torch.full((ns,), 3, dtype=torch.int64, device=dev)
        cnt_[0] = 2
        cnt_[-1] = 2
        rp_s = torch.zeros(ns + 1, dtype=torch.int64, device=dev)
        rp_s[1:] = torch.cumsum(cnt_, 0)
        cols_ = torch.stack([r_ - 1, r_, r_ + 1], 1).reshape(-1)
        vals_ = torch.tensor([0.5, -1.0, 0.5], dtype=torch.float64, device=dev).repeat(ns)
        keep_ = (cols_ >= 0) & (cols_ < ns)
        ci_s = cols_[keep_].to(torch.int32).contiguous()
        va_s = vals_[keep_].contiguous()
        del r_, cnt_, cols_, vals_, keep_
        for rep_i in range(2):
            b0 = torch.cuda.Event(enable_timing=True)
            b1 = torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            p = B.Plan(ns, rp_s, ci_s, va_s, args.eps_tol, stream=stream)
            p.run_only()
            b1.record(stream)
            torch.cuda.synchronize()
            ss = p.stats()
            p.close()
        Ns, Ms = int(ss["N"]), int(ss["M"])
        ty = [i for i in range(2, Ms + 1) if ss["taylor_numeric_ms"][i] > 0]
        tyb = sum(float(ss["taylor_numeric_bytes"][i]) for i in ty)
        tym = sum(float(ss["taylor_numeric_ms"][i]) for i in ty)
        config_s = {"workload": f"config S: 0.5 tridiag(1,-2,1), n = 2^25 (2^26 does not fit in 178 GB)",
                    "M": Ms, "N": Ns, "nnz_E": int(ss["nnz_out"]), "ms_expm": b0.elapsed_time(b1),
                    "phase_ms": {"plan": float(ss["ms_plan"]), "taylor": float(ss["ms_taylor"]),
                                 "squaring": float(ss["ms_squaring"]), "finalize": float(ss["ms_finalize"])},
                    "taylor_kernels_ms": tym, "taylor_kernels_compulsory_gbs": tyb / tym / 1e6 if tym else None,
                    "sq_kernel_ms": [float(x) for x in ss["sq_kernel_ms"][1:Ns + 1]]}
        del rp_s, ci_s, va_s
        B.sexpm_release_cache()

    # ---------------- the CPU sample on the GPU (same work as cpu_baseline / reference) ------
    same_sample = None
    if world == 1:
        Hs, gs = sample_config(args)
        rs_ = [torch.from_numpy(a).to(dev) for a in (Hs.rowptr, Hs.col, Hs.val)]
        ts = []
        for rep_i in range(4):
            b0 = torch.cuda.Event(enable_timing=True)
            b1 = torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            p = B.Plan(Hs.n, *rs_, args.eps_tol, stream=stream, **opts)
            p.run_only()
            b1.record(stream)
            torch.cuda.synchronize()
            p.close()
            if rep_i:
                ts.append(b0.elapsed_time(b1))
        same_sample = {"workload": f"config-{args.config} law on a {gs}x{gs} grid (n={Hs.n})",
                       "gpu_ms": min(ts), "gpu_e_per_s": 1000.0 / min(ts)}

    # ---------------- roofline of the dominant kernel ----------------
    import math
    sq_ms = [float(st["sq_kernel_ms"][i]) for i in range(1, N + 1)]
    sym = int(st["sq_sym_used"]) == N and N > 0
    # algorithmic flops of the squaring kernel: 2 per product of T T (sq_fmas = products +
    # nnz(T)); the symmetric kernel K3s computes the products with j >= r only -- for a
    # symmetric pattern exactly (products + nnz(T)) / 2 = sq_fmas / 2 of them
    sq_fl = [(1.0 if sym else 2.0) * float(st["sq_fmas"][i]) for i in range(1, N + 1)]
    sq_asm = [float(st["sq_assemble_ms"][i]) for i in range(1, N + 1)]
    ty_idx = [i for i in range(2, int(st["M"]) + 1) if st["taylor_numeric_ms"][i] > 0]
    ty_ms = [float(st["taylor_numeric_ms"][i]) for i in ty_idx]
    ty_by = [float(st["taylor_numeric_bytes"][i]) for i in ty_idx]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic_db = {}
    tp = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(tp):
        traffic_db = json.load(open(tp))
    if sum(sq_ms) >= sum(ty_ms) and sq_ms:
        dur = sum(sq_ms) / len(sq_ms) / 1e3
        ach = sum(sq_fl) / len(sq_fl) / dur / 1e12
        kname = "k_numeric_bsrm" if int(st["sq_bsr_blocks"][1]) > 0 else "k_numeric_paged"
        if sym:
            kname = "k_numeric_bsrm_sym"
        tr = traffic_db.get(kname)
        roof = {"kernel": f"{kname} (squaring SpGEMM + 2T + filter classify"
                          + (", output blocks J >= I of the symmetric T~)" if sym else ")"), "bound": "alu",
                "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP64_PEAK_TFLOPS,
                "traffic": tr["dram_bytes"] if tr and args.config == 5 else None,
                "traffic_launch": tr["launch"] if tr and args.config == 5 else None,
                "traffic_compulsory_bytes": float(st["sq_numeric_bytes"][1]),
                # the block kernel multiplies whole 8x8 blocks (zeros included): executed fp64
                # work (2 x 512 per block product) per launch, beside the algorithmic count
                "executed_fp64_tflops": (sum(1024.0 * float(st["sq_block_products"][i]) for i in range(1, N + 1))
                                         / len(sq_ms) / dur / 1e12),
                "peak_source": "measured on this GPU before the timed steps: sexpm_fp64_peak DFMA chains "
                               f"({FP64_PEAK_TFLOPS:.2f} TF/s; DMMA m8n8k4 {fp64_peak['dmma_tflops']:.2f} TF/s, "
                               "the instruction the kernel issues)",
                "dmma_peak": fp64_peak["dmma_tflops"],
                "launches_per_step": len(sq_ms), "avg_launch_ms": dur * 1e3,
                "symmetric_path": sym,
                # the full product's flops (2 sq_fmas) over K3s + K3c + K3a: the rate the
                # symmetric path delivers T~ at, for comparison with the full kernel
                "full_product_equiv_tflops": (sum(2.0 * float(st["sq_fmas"][i]) for i in range(1, N + 1))
                                              / (sum(sq_ms) + sum(sq_asm)) / 1e9) if sym else None,
                "assemble_ms": sq_asm if sym else None,
                "hbm_gbs_compulsory": sum(float(st["sq_numeric_bytes"][i]) for i in range(1, N + 1)) / len(sq_ms) / dur / 1e9}
    elif ty_ms:
        dur = sum(ty_ms) / len(ty_ms) / 1e3
        ach = sum(ty_by) / len(ty_by) / dur / 1e9
        tr = traffic_db.get("k_taylor_dia")
        roof = {"kernel": "k_taylor_dia (Taylor term S H0 / i + filter classify)", "bound": "hbm",
                "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "traffic": tr["dram_bytes"] if tr and args.config == 5 else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "launches_per_step": len(ty_ms), "avg_launch_ms": dur * 1e3}
    else:
        roof = None

    sq_total_ms = float(sum(st["sq_ms"][1:N + 1]))
    line = {
        "metric": METRIC, "value": value, "unit": "e^H/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, BASELINE.json config law)",
        "config": {"workload": f"BASELINE config {args.config}: 2D Dirichlet heat 1449x1449 r=0.5"
                   if args.config == 5 else f"BASELINE config {args.config}",
                   "n": n, "nnz_H": int(H.nnz), "eps_tol": args.eps_tol, "plan_norm": args.plan_norm,
                   "M": int(st["M"]), "N": N, "M_eff": int(st["M_eff"]), "nnz_E": int(st["nnz_out"]),
                   "parallelism": f"rows{world}", "l2": "flushed (256 MB write) between timed steps; working set >> L2"},
        "expm_wall_s": ms_per_step / 1e3,
        "squarings_per_s": (N / (sq_total_ms / 1e3)) if N and sq_total_ms > 0 else None,
        "phase_ms": {"plan": float(st["ms_plan"]), "taylor": float(st["ms_taylor"]),
                     "squaring": float(st["ms_squaring"]), "finalize": float(st["ms_finalize"]),
                     "order_host_thread": float(st["ms_order_host"]),
                     "order_wait": float(st["ms_order_wait"])},
        "roofline": roof,
        "steps_detail": [{"ms": times[j], "retries": int(stats[j]["retries"]),
                          "taylor_ms": float(stats[j]["ms_taylor"]),
                          "sq_numeric_ms": [float(x) for x in stats[j]["sq_numeric_ms"][1:N + 1]],
                          "sq_kernel_ms": [float(x) for x in stats[j]["sq_kernel_ms"][1:N + 1]],
                          "sq_first_ms": [float(x) for x in stats[j]["sq_first_ms"][1:N + 1]],
                          "sq_fallback_rows": [int(x) for x in stats[j]["sq_fallback_rows"][1:N + 1]],
                          "cache_misses": int(stats[j]["cache_misses"])}
                         for j in range(len(stats))],
        "gpu_launches": int(launches),
        "e2e": e2e,
        "apply": apply_res,
        "n2_filter_off": n2,
        "n3_reorder": n3,
        "n4_graph": n4,
        "other_configs": others,
        "config_s": config_s,
        "same_sample": same_sample,
        "fp64_peak_measured": fp64_peak,
    }
    if rank == 0:
        line["clocks"] = clk.summary()
        if world == 1 and not args.no_cpu_baseline:
            v, cores, sample, dt = cpu_oracle_sample(args)
            line["cpu_baseline"] = {"value": v, "unit": "e^H/s", "cores": cores, "kind": "oracle",
                                    "sample": sample, "sample_seconds": dt}
            if same_sample:
                same_sample["cpu_s"] = dt
                same_sample["gpu_over_cpu"] = dt * 1000.0 / same_sample["gpu_ms"]
        print(json.dumps(line, default=lambda o: float(o) if hasattr(o, "__float__") else str(o)),
              flush=True)
    if comm is not None:
        B.sexpm_nccl_comm_destroy(comm)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Benchmark: training chars/s of the paper's 4096-d mLSTM step (seq 256, 256 rows/GPU, mixed fp16/fp32
with dynamic loss scaling) on N B200s, data parallel (BASELINE.json `metric`, configs[2]).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C1|C2|C3|C4|C5] [--weight-norm]
  N > 1: python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Rank 0 prints ONE JSON line.  `value` = N*B*T / (max over ranks of the CUDA-event time of K steps)/K,
inputs resident in HBM.  `e2e` = the same metric through mlstm_train_step_host (pinned host bytes
H2D + result D2H inside the timed region).  `roofline` = the dominant GEMM phase's algorithmic
FLOP/s vs MEASURED_PEAKS.json.  `cpu_baseline` = the fp64 oracle on a bounded sample (rank 0, N=1).
--impl reference times that oracle alone (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

if __name__ == "__main__":  # oracle / numpy threads = all host cores (set before numpy loads)
    _n = str(len(os.sched_getaffinity(0)))
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(_v, _n)

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training chars/sec (4096-d mLSTM, seq 256) at 1/2/4/8 B200; tensor-pipe %"
CONFIGS = {
    # name: (h, e, B per GPU, T, description)
    "C1": (64, 64, 4, 16, "tiny mLSTM h=64 e=64, seq 16, batch 4/GPU"),
    "C2": (1024, 64, 128, 64, "mLSTM h=1024 e=64, seq 64, batch 128/GPU"),
    "C3": (4096, 64, 256, 256, "paper model: mLSTM h=4096 e=64, seq 256, batch 256/GPU, fp16/fp32 mixed, "
                               "dynamic loss scaling"),
    "C4": (4096, 64, 4096, 256, "large batch: mLSTM h=4096 e=64, seq 256, 4096 rows/GPU as 4 x 1024-row "
                                "micro-batches (global batch 32768 at 8 GPUs), fp16/fp32 mixed"),
    "C5": (8192, 64, 128, 256, "8192-d mLSTM e=64, seq 256, batch 128/GPU, fp16/fp32 mixed, lr0 7.8e-4 (P:240)"),
    "C5-256": (8192, 64, 256, 256, "8192-d mLSTM e=64, seq 256, batch 256/GPU (P:240's memory-bound 96/GPU on "
                                   "V100; B200 fits 256 without recompute), fp16/fp32 mixed, lr0 7.8e-4"),
}
LR0 = {"C5": 7.8e-4, "C5-256": 7.8e-4}  # the 8192-d model's square-root-scaled learning rate
MICRO_BATCH = {"C4": 1024}
DEVSTATE_BYTES = 56  # the device scalar block the step copies back (loss, alpha, lr, skip, it, tau)


def flops_per_char(h, e):
    """6 (5h^2 + 5he + 256h) -- fwd, dW and dX of every matmul."""
    return 6.0 * (5 * h * h + 5 * h * e + 256 * h)


def phase_flops(h, e, B, T):
    """Algorithmic FLOPs of each GEMM phase of one step (per rank)."""
    BT = B * T
    return {
        "fwd_rec": 2.0 * BT * 5 * h * h,                                   # W_mh h, W_h m per char
        "bwd_rec": 2.0 * BT * 5 * h * h - 2.0 * B * h * h + 2.0 * BT * 256 * h,  # dZ W_h, dA W_mh (t>0),
                                                                            # dY W_dec (folded into B2)
        "wgrad": 2.0 * BT * (5 * h * h + 5 * h * e + 256 * h),             # dW_h, dW_mh, dW_x, dW_mx, dW_dec
        "decoder": 2.0 * BT * 256 * h,
    }


def kernel_table(h, e, B, T, kind):
    """The kernels of each GEMM phase of one step: name -> (phase, launches per step, algorithmic FLOP per
    launch).  Names match profiles/ncu_kernel_share.json (tools/kernel_share.py).  kind: the
    recurrence implementation (mlstm_recurrence_kind: 0 per-timestep, 1 persistent, 3 persistent
    forward + per-timestep BPTT)."""
    pf = phase_flops(h, e, B, T)
    tab = {
        "gemm_tc2_kernel<512,EpiWgrad,MN>": ("wgrad", 3, 2.0 * B * T * (5 * h * h + 256 * h) / 3),
        "gemm_tc2p_kernel<256,EpiY>": ("decoder", 1, 2.0 * B * T * 256 * h),
    }
    if kind in (1, 3):
        tab["fwd_recur_kernel"] = ("fwd_rec", 1, pf["fwd_rec"])
    else:
        tab["gemm_tc1s_kernel<4,EpiF1IO>"] = ("fwd_rec", T, 2.0 * B * h * h)        # a_t = H_{t-1} W_mh^T
        tab["gemm_tc2_kernel<256,EpiF2IO>"] = ("fwd_rec", T, 2.0 * B * 4 * h * h)   # z_t = M_t W_h^T (+ one-hot seg)
    if kind == 1:
        tab["bwd_recur_kernel"] = ("bwd_rec", 1, pf["bwd_rec"])
    else:  # the backward reads the weights MN-major (",BMN"): dM_t = dZ_t W_h; dA_t W_mh + dY_{t-1} W_dec
        tab["gemm_tc1s_kernel<4,EpiB1IO,BMN>"] = ("bwd_rec", T, 2.0 * B * 4 * h * h)
        tab["gemm_tc1s_kernel<4,EpiB2,BMN>"] = ("bwd_rec", T - 1, 2.0 * B * (h + 256) * h)
    return tab


def kernel_shares(kind):
    """phase -> {kernel: share of the phase's kernel time}."""
    out = {}
    try:
        tab = json.load(open(os.path.join(ROOT, "profiles", "ncu_kernel_share.json")))["per_timestep"]["phases"]
        out = {ph: {k: v["share"] for k, v in ks.items()} for ph, ks in tab.items()}
    except (OSError, ValueError, KeyError):
        pass
    if kind in (1, 3):  # one kernel per persistent recurrence phase
        out["fwd_rec"] = {"fwd_recur_kernel": 1.0}
    if kind == 1:
        out["bwd_rec"] = {"bwd_recur_kernel": 1.0}
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": float(np.median(pw)) if pw else None}


def host_info():
    """CPU model and the BLAS numpy links (the oracle's matmul library)."""
    cpu = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = "unknown"
    try:
        cfg = np.__config__.CONFIG["Build Dependencies"]["blas"]
        blas = f"{cfg.get('name')} {cfg.get('version', '')}".strip()
    except Exception:
        pass
    return cpu, blas


class OracleSampler:
    """The fp64 oracle as it stands, timed on a bounded sample of the same workload: same h and e, the
    oracle batch of SURVEY 8(d) (B = 8 rows), window length sized so one sample is ~seconds_hint of
    CPU work: forward, BPTT and Adam."""

    def __init__(self, h, e, seconds_hint=15.0, B=8):
        from oracle import mlstm_oracle as O
        from synth import bytestream
        self.O, self.h, self.e, self.B = O, h, e, B
        self.cores = len(os.sched_getaffinity(0))
        self.cpu, self.blas = host_info()
        self.P = O.init_params(h, e, 0x5EED)
        self.theta = O.flatten(self.P)
        # Per timestep the oracle streams every fp64 weight matrix a few times, so its cost is nearly
        # flat in the row count: calibrate on a short window, then size the window.
        by = bytestream.window(np.arange(B), 0, 4)
        z = np.zeros((B, h))
        t0 = time.perf_counter()
        O.loss_and_grads(self.P, by, z, z)
        per_step = (time.perf_counter() - t0) / 4
        self.T = int(max(4, min(256, seconds_hint / max(per_step, 1e-4))))
        self.by = bytestream.window(np.arange(B), 0, self.T)
        self.seconds = None

    def run(self):
        O, B, h = self.O, self.B, self.h
        z = np.zeros((B, h))
        t0 = time.perf_counter()
        _, g, _, _ = O.loss_and_grads(self.P, self.by, z, z)
        st = O.AdamState(np.zeros_like(self.theta), np.zeros_like(self.theta))
        O.adam_apply(self.theta, O.flatten(g), st, 3e-3)
        dt = time.perf_counter() - t0
        self.seconds = dt
        return {"value": B * self.T / dt, "unit": "chars/s", "cores": self.cores, "kind": "oracle",
                "cpu": self.cpu, "blas": self.blas, "sample_rows": B, "sample_T": self.T, "seconds": round(dt, 2),
                "sample": f"fp64 NumPy oracle, h={h} e={self.e}, {B} rows x T={self.T} window (forward, BPTT, "
                          f"Adam), {dt:.1f} s on {self.cores} host threads ({self.cpu}; BLAS {self.blas})"}


def cpu_baseline(h, e, seconds_hint=15.0):
    return OracleSampler(h, e, seconds_hint).run()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    h, e, B, T, desc = CONFIGS[args.config]
    # each "step" is one bounded sample of the workload on the host cores; the whole run stays
    # within a few minutes
    sampler = OracleSampler(h, e, seconds_hint=min(args.ref_seconds, 150.0 / (args.warmup + args.steps)))
    vals, secs = [], []
    for i in range(args.warmup + args.steps):
        r = sampler.run()
        if i >= args.warmup:
            vals.append(r["value"])
            secs.append(r["seconds"])
    v = float(np.median(vals))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "chars/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.median(secs)) * 1e3,  # the wall time of one bounded sample (a "step" here)
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "global_batch": B * args.gpus, "seq_len": T, "parallelism": f"dp{args.gpus}",
                   "sample": f"each step = {sampler.B} rows x T={sampler.T} of this workload on the host cores"},
        "cpu_baseline": {**r, "value": v},
        "e2e": {"value": v, "unit": "chars/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)  # median over 50 steps
    ap.add_argument("--warmup", type=int, default=5)  # 5 warm-up steps
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--weight-norm", action="store_true",
                    help="weight-normalised LSTM matrices (P:150; SURVEY NEXT #1)")
    ap.add_argument("--recurrence", type=int, default=0, choices=[0, 1, 2, 3],
                    help="mlstm_config.recurrence: 0 library default, 1 persistent dataflow kernels, 2 per-timestep, "
                         "3 persistent forward + per-timestep BPTT")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_1808_01371_b200 as M
    from synth import bytestream

    rank, local, world = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h, e, B, T, desc = CONFIGS[args.config]
    if args.weight_norm:
        desc += "; weight-normalised W_mx, W_mh, W_x, W_h (P:150)"
    cfg = M.mlstm_default_config(hidden=h, embed=e, batch=B, seq_len=T, precision=M.MLSTM_MIXED,
                                 micro_batch=MICRO_BATCH.get(args.config, 0),
                                 weight_norm=1 if args.weight_norm else 0, recurrence=args.recurrence)
    if args.config in LR0:
        cfg.lr0 = LR0[args.config]
    nid = None
    if world > 1:
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(M.mlstm_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        nid = bytes(t.cpu().numpy().tobytes())
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        model = M.MLSTM(cfg, rank=rank, world=world, nccl_id=nid, stream=stream)
    nsteps = args.warmup + args.steps
    rows = np.arange(rank * B, (rank + 1) * B)
    windows = bytestream.windows(rows, 0, nsteps + (0 if args.no_e2e else args.steps), T)
    dev = torch.from_numpy(windows[:nsteps].copy()).to(f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])

    # phase events are part of the step's graphs from the first warm-up step on (profiling enabled
    # before it), so nothing is re-recorded in the timed region; re-enabling only resets the phase
    # accumulators, which then sum exactly the K timed steps
    model.profile(True)
    for i in range(args.warmup):
        model.train_step(dev[i])
    launches = model.launches_per_step()
    model.profile(True)
    barrier()
    # timed region: K steps (one CUDA event per step on the step's stream)
    clocks = ClockSampler(local)
    clocks.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    results = []
    for k, i in enumerate(range(args.warmup, nsteps)):
        results.append(model.train_step(dev[i]))
        evs[k + 1].record(stream)
    barrier()
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[-1])
    step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    med = float(np.median(step_ms))
    if world > 1:
        tt = torch.tensor([ms, med], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, med = float(tt[0].item()), float(tt[1].item())
    ms_step = ms / args.steps
    value = world * B * T / (ms_step / 1e3)
    phases = {k: (v[0] / args.steps, v[1]) for k, v in model.phase_times().items()}

    # end to end through the public host entry point (pinned host bytes in, result struct out)
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(windows[nsteps:].copy()).pin_memory()
        host = pinned.numpy()
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            model.train_step_host(host[i])
        t1.record(stream)
        barrier()
        ems = t0.elapsed_time(t1)
        if world > 1:
            tt = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": world * B * T / (ems / args.steps / 1e3), "unit": "chars/s",
               "h2d_bytes_per_step": B * (T + 1), "d2h_bytes_per_step": DEVSTATE_BYTES}

    if rank != 0:
        return
    burst, sustained, hbm, src = load_peaks()
    pf = phase_flops(h, e, B, T)
    gem = {k: phases[k] for k in pf if k in phases}
    # dominant kernel: phase time (live events) x the kernel's share of that phase (committed ncu
    # launch list, tools/kernel_share.py); per-launch time = that / its launches per step
    kind = M.lib().mlstm_recurrence_kind(model.ctx)
    ktab, shares = kernel_table(h, e, B, T, kind), kernel_shares(kind)
    kt = {}
    for k, (ph, nl, fl) in ktab.items():
        sh = shares.get(ph, {}).get(k)
        if ph in gem and sh is not None:
            kt[k] = (gem[ph][0] * sh, nl, fl, ph, sh)
    dom = max(kt, key=lambda k: kt[k][0])
    kms, nl, fl, ph, sh = kt[dom]
    us_launch = kms / nl * 1e3
    achieved = fl / (us_launch / 1e6) / 1e12
    traffic = None
    try:  # measured DRAM bytes per launch of this kernel (committed ncu --set full capture)
        tj = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tj.get(args.config, {}).get(ph, {}).get("kernels", {}).get(dom)
    except (OSError, ValueError):
        pass
    roof = {"bound": "tensor", "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
            "frac": achieved / sustained, "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
            "peak_source": f"{src} bf16_tflops_sustained (fp16 dense = bf16 dense rate)",
            "kernel": dom, "launches_per_step": nl, "gflop_per_launch": round(fl / 1e9, 3),
            "us_per_launch": round(us_launch, 2),
            "how": f"{ph} phase {gem[ph][0]:.3f} ms/step (CUDA events in the step graph over the timed steps) "
                   f"x share {sh:.3f} (ncu launch list, profiles/ncu_kernel_share.json) / {nl} launches"}
    # every GEMM phase against the same sustained peak, and the recurrences also against HBM: every
    # timestep re-streams the recurrent weights (fp16) and moves its stash rows (10h^2
    # weight bytes per timestep and direction pair; ~48h stash bytes per row per timestep)
    roof_phases = {k: {"tflops": round(pf[k] / (gem[k][0] / 1e3) / 1e12, 1),
                       "frac": round(pf[k] / (gem[k][0] / 1e3) / 1e12 / sustained, 3),
                       "ms": round(gem[k][0], 3)} for k in gem if gem[k][0] > 0}
    for k, wbytes in (("fwd_rec", 2.0 * 5 * h * h), ("bwd_rec", 2.0 * (5 * h * h + 256 * h))):
        if k in roof_phases:
            gbs = T * (wbytes + 24.0 * h * B) / (gem[k][0] / 1e3) / 1e9
            roof_phases[k]["hbm_gbs"] = round(gbs, 1)
            roof_phases[k]["hbm_frac"] = round(gbs / hbm, 3)
    whole = flops_per_char(h, e) * world * B * T / (ms_step / 1e3) / 1e12 / world
    line = {
        "metric": METRIC, "value": value, "unit": "chars/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_median": med, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16 (fp32 accumulate, fp32 masters)", "data": "synthetic",
        "config": {"workload": desc, "global_batch": world * B, "seq_len": T, "parallelism": f"dp{world}",
                   "recurrence": {1: "persistent dataflow kernels", 3: "persistent forward, per-timestep BPTT"}.get(
                       kind, "per-timestep GEMM launches"),
                   "l2": "no flush: per-step working set (~11 GB) >> 126 MB L2"},
        "roofline": roof, "roofline_phases": roof_phases,
        "step_tflops_per_gpu": whole, "step_frac_of_sustained_peak": whole / sustained,
        "phases_ms_per_step": {k: round(v[0], 4) for k, v in phases.items()},
        "phases_from": "CUDA events inside the step's graphs, summed over the K timed steps",
        "clocks": clk, "e2e": e2e, "gpu_launches": launches * args.steps,
        "loss_first_last": [results[0]["loss_nats"], results[-1]["loss_nats"]],
        "skipped_steps": int(sum(r["skipped"] for r in results)),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(h, e)
    print(json.dumps(line), flush=True)
    model.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

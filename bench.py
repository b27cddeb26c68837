"""Benchmark: spark fitness evaluations/s and ms/generation of the B200
MGFWA engine on BASELINE.json's configs[1] (C2: MLP-weights black box
784-32-10, S = 1024 synthetic samples, B = 1, mu = 5 fireworks x lambda = 300
sparks, M = 3 guides).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c1|c2|c3|c4|c5] [--scaling weak|strong]

A "step" is one MGFWA generation (the body of run()'s loop,
engine.cpp:359-417) on synthetic data.  value = whole-job evaluations per
second, device-timed with CUDA events on the engine's stream over exactly K
generations (max over ranks).  e2e = the same metric through the one-shot
C-ABI run() drop-in (mgfwa_run_once) with host buffers in and out.
Multi-GPU (torchrun, N ranks): weak scaling by default — the population grows
to N x mu fireworks, each rank owns mu of them, and one in-place NCCL
all-gather of the selected fireworks per generation keeps the population
state replicated; ``--scaling strong`` splits the workload's
own mu fireworks over the ranks instead (C5: 64 fireworks, 8 per GPU at N=8).  ``--impl reference`` times the compiled reference
(oracle/_ref, /root/reference/proj/src/engine.cpp run()) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

WORKLOADS = {
    # BASELINE.json configs[1] (headline)
    "c2": dict(desc="C2 MLP-weights 784-32-10, S=1024, B=1, mu=5, lambda=300, M=3", kind="mlp", D=25450,
               B=1, mu=5, lam=300, M=3, lo=-1.0, hi=1.0, in_dim=784, hidden=32, out_dim=10, samples=1024),
    # configs[0]
    "c1": dict(desc="C1 sphere D=30, B=1, mu=5, lambda=30, M=3", kind="sphere", D=30, B=1, mu=5, lam=30, M=3,
               lo=-10.0, hi=10.0),
    # configs[2]: LeNet-5 on 28x28 synthetic samples
    "c3": dict(desc="C3 LeNet-5 (conv6-conv16-120-84-10), S=1024, B=1, mu=5, lambda=300, M=3", kind="lenet",
               D=61706, B=1, mu=5, lam=300, M=3, lo=-1.0, hi=1.0, samples=1024),
    # configs[4]: large population, MLP 784-256-10 (weak-scaling firework shards)
    "c5": dict(desc="C5 MLP-weights 784-256-10, S=1024, B=1, mu=64, lambda=1024, M=3", kind="mlp", D=203530,
               B=1, mu=64, lam=1024, M=3, lo=-1.0, hi=1.0, in_dim=784, hidden=256, out_dim=10, samples=1024),
    # configs[3]
    "c4": dict(desc="C4 Rastrigin D=1e5, B=1, mu=5, lambda=30, M=3", kind="rastrigin", D=100000, B=1, mu=5,
               lam=30, M=3, lo=-5.12, hi=5.12),
}
FLOP_PER_EVAL_C2 = 2 * 1024 * (784 * 32 + 32 * 10)  # 52,035,584
LENET_FLOP_PER_SAMPLE = 833_040  # conv1 117,600 + conv2 240,000 + fc 58,920 MAC, x2


def flop_per_eval(w):
    """Algorithmic FLOP of one candidate evaluation."""
    if w["kind"] == "lenet":
        return LENET_FLOP_PER_SAMPLE * w["samples"]
    return 2 * w["samples"] * (w["in_dim"] * w["hidden"] + w["hidden"] * w["out_dim"])


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def ncu_traffic(kernel_prefix: str):
    """DRAM bytes (read + write) per launch of a kernel from the latest
    committed `ncu --set full` capture under profiles/ (None if absent)."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_full_hot_kernels.json")), reverse=True):
        with open(path) as f:
            for k in json.load(f):
                if kernel_prefix in k.get("kernel", ""):
                    def mb(s):
                        v, unit = s.split()
                        return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
                    try:
                        return {"bytes": mb(k["dram__bytes_read.sum"]) + mb(k["dram__bytes_write.sum"]),
                                "source": os.path.relpath(path, ROOT)}
                    except (KeyError, ValueError):
                        return None
    return None


def make_objective(P, w):
    if w["kind"] == "mlp":
        return P.MlpWeights(w["in_dim"], w["hidden"], w["out_dim"], w["samples"], 1)
    if w["kind"] == "lenet":
        return P.LeNet(w["samples"], 1)
    return {"sphere": P.Sphere(), "rastrigin": P.Rastrigin(), "ackley": P.Ackley()}[w["kind"]]


class stdout_to_stderr:
    """fd-level redirect of stdout to stderr (native libraries print there)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def make_config(P, w, max_evals):
    return P.MgfwaConfig(batches=w["B"], fireworks=w["mu"], sparks_per_firework=w["lam"],
                         guides_per_firework=w["M"], boosts=[1.0, 2.0, 4.0][: w["M"]],
                         max_evaluations=max_evals)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                pass

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                for n, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _ref_desc(O, w):
    kind = {"mlp": O.OBJ_MLP_WEIGHTS, "lenet": O.OBJ_LENET, "sphere": O.OBJ_SPHERE,
            "rastrigin": O.OBJ_RASTRIGIN, "ackley": O.OBJ_ACKLEY}[w["kind"]]
    return O.ObjectiveDesc(kind=kind, in_dim=w.get("in_dim", 784), hidden=w.get("hidden", 32),
                           out_dim=w.get("out_dim", 10), samples=w.get("samples", 1024))


def cpu_reference_generation(w, seed: int, workers: int):
    """Reference CPU throughput on the host cores via the compiled reference
    (oracle/_ref).  C1/C2/C4: one full generation, run() with budget
    init + 1 wave.  C3/C5, whose CPU generations take minutes to hours
    (SURVEY.md §8(d)): batched_apply() of a bounded sample of candidate rows
    (fitness only, the dominant reference cost), extrapolated as evals/s.
    Returns (evals, seconds, sample description)."""
    import oracle as O

    ref = O.Reference()
    desc = _ref_desc(O, w)
    if w["kind"] == "lenet" or w["D"] > 100000:
        n = max(workers, 1) * (2 if w["kind"] == "lenet" else 1)
        rows = np.random.default_rng(seed).uniform(w["lo"], w["hi"], size=(n, w["D"])) * 0.05
        t = time.perf_counter()
        ref.batched_apply(desc, rows[None], workers=workers)
        return n, time.perf_counter() - t, f"batched_apply() of {n} candidate rows (fitness only)"
    cfg = O.Config(batches=w["B"], fireworks=w["mu"], sparks_per_firework=w["lam"], guides_per_firework=w["M"],
                   boosts=[1.0, 2.0, 4.0][: w["M"]],
                   max_evaluations=w["B"] * w["mu"] + w["B"] * w["mu"] * (w["lam"] + w["M"]))
    lo, hi = np.full(w["D"], w["lo"]), np.full(w["D"], w["hi"])
    t = time.perf_counter()
    r = ref.run(cfg, lo, hi, desc, seed, workers=workers)
    return r.evaluations_used, time.perf_counter() - t, "mgfwa::run() of one generation (init + 1 wave)"


def run_reference_arm(args, w):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    evals, secs, steps = 0, 0.0, 0
    t0 = time.perf_counter()
    what = ""
    for _ in range(args.warmup):  # bounded warm-up
        cpu_reference_generation(w, 1000, cores)
        if time.perf_counter() - t0 > 30:
            break
    t1 = time.perf_counter()
    for k in range(args.steps):
        e, s, what = cpu_reference_generation(w, k, cores)
        evals += e
        secs += s
        steps += 1
        if time.perf_counter() - t1 > 150:  # keep the arm within a few minutes
            break
    v = evals / secs
    line = {"metric": "spark fitness evals/sec", "value": v, "unit": "evals/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w["desc"], "budget_per_step": "init + 1 generation"}, "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "evals/s", "cores": cores, "kind": "reference",
                             "sample": f"{steps} x {what}, EvalBackend::data_parallel({cores})"},
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = mu fireworks per rank (default); strong = the workload's mu "
                         "fireworks split over the ranks (e.g. C5: 64 fireworks, 8 per GPU at N=8)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--distributed", action="store_true",
                    help="take the torch.distributed / NCCL sharded code path even at N = 1 "
                         "(a 1-rank communicator; used to test the multi-GPU path on one GPU)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard-mode", choices=["firework", "replica"], default="firework",
                    help="N>1: firework = fireworks split over the ranks, selected state all-gathered each "
                         "generation; replica = batches x N, each rank owns whole batches, only the loser count "
                         "is exchanged (weak scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]

    if args.impl == "reference":
        run_reference_arm(args, w)
        return

    import torch

    world, rank, local = dist_env()
    sharded = world > 1 or args.distributed
    if sharded:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))

        torch.cuda.set_device(local)
        with stdout_to_stderr():  # NCCL's version banner: keep stdout to the one JSON line
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
    else:
        torch.cuda.set_device(0)
    import paper_2501_03944_b200 as P

    dev = torch.cuda.current_device()
    stream = torch.cuda.Stream()
    obj = make_objective(P, w)
    space = P.SearchSpace.box(w["D"], w["lo"], w["hi"])
    # N > 1: weak scaling — the population grows to mu * N fireworks, each
    # rank owns mu of them (firework sharding), one in-place NCCL all-gather
    # of the selected fireworks per generation.
    wn = dict(w)
    replica = args.shard_mode == "replica"
    if replica:
        wn["B"] = w["B"] * world
    elif args.scaling == "weak":
        wn["mu"] = w["mu"] * world
    elif (w["B"] * w["mu"]) % world != 0:
        raise SystemExit(f"--scaling strong needs B*mu divisible by the rank count ({w['B'] * w['mu']} % {world})")
    eng = P.Engine(make_config(P, wn, 1 << 62), space, obj, seed=0, device=dev, rank=rank, world=world,
                   shard_mode=args.shard_mode)
    if sharded:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(P.Engine.nccl_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(uid, 0)
        with stdout_to_stderr():
            eng.attach_nccl(bytes(uid.cpu().numpy().tobytes()))
    eng.set_stream(stream.cuda_stream)
    eng.initialize()
    kpg = eng.kernels_per_generation()
    eng.enqueue(args.warmup)
    eng.sync()
    before = eng.counters()["evaluations_used"]

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if sharded:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        with torch.cuda.stream(stream):
            start.record(stream)
            eng.enqueue(args.steps)
            end.record(stream)
        torch.cuda.synchronize()
    if sharded:
        torch.distributed.barrier()
    eng.sync()
    ms = start.elapsed_time(end)
    # evaluations_used is the population-wide counter, identical on every rank
    evals = eng.counters()["evaluations_used"] - before
    if sharded:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_max, evals_total = float(t[0]), float(evals)
    else:
        ms_max, evals_total = ms, float(evals)

    # dominant kernel: spark fitness (tcgen05 GEMM) timed alone, CUDA events
    fit_ms, units = eng.time_fitness(20)
    pk, pk_kind = peaks()
    if w["kind"] in ("mlp", "lenet"):
        fpe = flop_per_eval(w)
        achieved = fpe * units / (fit_ms * 1e-3) / 1e12
        if w["kind"] == "mlp":
            kname = f"k_mlp_fitness<{w['hidden']}> (tcgen05.mma kind::f16, TMA, TMEM)"
            tr = ncu_traffic(f"k_mlp_fitness<{w['hidden']}")
            opb = units * w["D"] * 2 + w["samples"] * w["in_dim"] * 2
        else:
            kname = "k_lenet_conv + k_lenet_fc (mma.sync m16n8k16 bf16, weights staged in smem)"
            tc, tf = ncu_traffic("k_lenet_conv"), ncu_traffic("k_lenet_fc")
            tr = {"bytes": tc["bytes"] + tf["bytes"], "source": tc["source"]} if tc and tf else None
            # + the pooled conv2 activations through the HBM scratch (bf16 x 400, written + read)
            opb = units * w["D"] * 2 + w["samples"] * 784 * 2 + 2 * units * w["samples"] * 800
        roof = {"kernel": kname, "bound": "tensor",
                "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16_tflops"], "traffic": tr["bytes"] if tr else None,
                "traffic_source": tr["source"] if tr else None,
                "algorithmic_per_launch": f"{units} candidates x {fpe} FLOP; operand bytes {opb} (bf16 W + X)",
                "ms_per_launch": fit_ms, "peak_source": f"{pk_kind} bf16 burst (MEASURED_PEAKS.json)"}
    else:
        byts = units * w["D"] * 4 + w["B"] * w["mu"] * w["D"] * 4
        achieved = byts / (fit_ms * 1e-3) / 1e9
        roof = {"kernel": "k_explode_map (fused explode+map+fitness)", "bound": "hbm", "achieved": achieved,
                "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": None,
                "ms_per_launch": fit_ms, "peak_source": f"{pk_kind} hbm copy"}

    line = {"metric": "spark fitness evals/sec", "value": evals_total / (ms_max * 1e-3), "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "bf16" if w["kind"] in ("mlp", "lenet") else "f32", "data": "synthetic",
            "config": {"workload": w["desc"], "D": w["D"], "fireworks_total": wn["mu"] * wn["B"],
                       "parallelism": (f"batch replicas x{world} ({wn['B']} batches)" +
                                       (" + 8-byte NCCL all-reduce/gen" if world > 1 else "")) if replica else
                                      (f"firework-sharded x{world}" + (" + NCCL all-gather/gen" if world > 1 else "")),
                       "l2": "inputs larger than L2: spark matrix fp32+bf16 229 MB/generation > 126 MB"
                       if args.workload == "c2" else "n/a"},
            "gpu_launches": kpg * args.steps if kpg else 1,  # 1: the persistent small-problem loop
            "roofline": roof}
    line["clocks"] = clk.summary()
    # per-kernel device times of the generation's idempotent kernels on the
    # steady-state engine (CUDA events, back-to-back launches) with their
    # achieved HBM bandwidth against algorithmic bytes (GB/s
    # for generation and guiding); per rank's own fireworks.
    try:
        Fl = wn["B"] * wn["mu"] // world
        Dp4, nn = w["D"] * 4, w["kind"] in ("mlp", "lenet")
        top = -(-w["lam"] // 5)  # ceil(0.2 * lambda), the default guide fraction
        algo = {"explode": Fl * w["lam"] * w["D"] * (6 if nn else 4) + Fl * w["D"] * 4,
                "guides": Fl * (2 * top * Dp4 + w["M"] * w["D"] * (6 if nn else 4) + Dp4),
                "rank": Fl * w["lam"] * (4 if nn else 8) * 2,
                # winner row read + firework row written (every firework's winner a spark or
                # guide: the upper bound) + the spark fitness scan
                "select": Fl * (2 * w["D"] * 4 + w["lam"] * 4)}
        kb = {}
        for name in ("explode", "rank", "guides", "select"):
            kms, _ = eng.time_kernel(name, 10)
            kb[name] = {"us": 1e3 * kms, "algorithmic_bytes": algo[name],
                        "achieved_GBs": algo[name] / (kms * 1e-3) / 1e9,
                        "frac_hbm": algo[name] / (kms * 1e-3) / 1e9 / pk["hbm_gbs"]}
        if nn:
            for name in ("fitness", "guide_fitness"):
                kms, units_k = eng.time_kernel(name, 10)
                kb[name] = {"us": 1e3 * kms, "rows": units_k,
                            "achieved_TFLOPs": flop_per_eval(w) * units_k / (kms * 1e-3) / 1e12}
        line["kernel_breakdown"] = kb
    except Exception as ex:
        line["kernel_breakdown"] = {"error": str(ex)[:200]}

    if sharded and not args.no_e2e:
        # e2e at N GPUs through the public API: every rank holds its shard of
        # the engine (created from the host config / bounds) in the NCCL
        # clique; the timed region is run() (initialize + K generations with
        # the per-generation all-gather and the host syncs of the step loop)
        # and the D2H of the best; wall-clock per rank, max over ranks.
        import torch.distributed as dist

        cfg_e = make_config(P, wn, wn["B"] * wn["mu"] + args.steps * wn["B"] * wn["mu"] * (w["lam"] + w["M"]))

        # the engine shard and its NCCL communicator are set up once (like a
        # long-lived service); each timed run() re-initializes from the host
        # config and reads the best back
        e = P.Engine(cfg_e, space, obj, seed=7, device=dev, rank=rank, world=world, shard_mode=args.shard_mode)
        u = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            u.copy_(torch.frombuffer(bytearray(P.Engine.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(u, 0)
        with stdout_to_stderr():
            e.attach_nccl(bytes(u.cpu().numpy().tobytes()))

        def sharded_once():
            dist.barrier()
            t0 = time.perf_counter()
            e.run()
            e.best()
            used = e.counters()["evaluations_used"]
            dt = time.perf_counter() - t0
            tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return used, float(tt[0])

        try:
            sharded_once()  # warm (module load, workspace, NCCL first use)
            used, dt = sharded_once()
            B, D = wn["B"], w["D"]
            line["e2e"] = {"value": used / dt, "unit": "evals/s",
                           "h2d_bytes_per_step": 0,  # config and bounds copied at engine creation
                           "d2h_bytes_per_step": (B * D * 8 + B * 8) / args.steps,
                           "what": f"run() (initialize from the host config + {args.steps} generations, per-"
                                   f"generation NCCL {'loser-count all-reduce' if replica else 'all-gather'}) + "
                                   f"best() D2H on {world} GPUs, wall-clock max over "
                                   f"ranks; engine shard and communicator created once"}
        except Exception as ex:  # keep the device-timed line
            line["e2e"] = {"value": None, "unit": "evals/s", "error": str(ex)[:200]}
        e.close()

    if rank == 0 and not sharded and not args.no_e2e:
        # e2e: one-shot run() drop-in over host buffers (mgfwa_run_once):
        # budget = init + K generations; includes context setup, H2D of the
        # search bounds, the K generations and D2H of best/trace.
        import ctypes as C

        from paper_2501_03944_b200 import _capi as A

        cfg = make_config(P, w, w["B"] * w["mu"] + args.steps * w["B"] * w["mu"] * (w["lam"] + w["M"]))
        c, keep = cfg._c()
        sp, ob = space._c(), obj._c()
        B, D = w["B"], w["D"]
        bf, bp = np.empty(B), np.empty((B, D))
        cap = args.steps + 2
        te, tb, tw = np.zeros((B, cap), np.uint64), np.zeros((B, cap)), np.zeros((B, cap))
        cnt = A.mgfwa_counters_t()
        pdp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731

        def once():
            rc = A.lib().mgfwa_run_once(C.byref(c), C.byref(sp), C.byref(ob), 7, dev, pdp(bf), pdp(bp),
                                        te.ctypes.data_as(C.POINTER(C.c_uint64)), pdp(tb), pdp(tw), cap,
                                        C.byref(cnt))
            assert rc == 0, A.lib().mgfwa_last_error(None)

        once()  # warm (module load, first-touch)
        t = time.perf_counter()
        once()
        dt = time.perf_counter() - t
        line["e2e"] = {"value": cnt.evaluations_used / dt, "unit": "evals/s",
                       "h2d_bytes_per_step": (2 * D * 8 + 8 * 12) / args.steps,
                       "d2h_bytes_per_step": (B * D * 8 + B * 8 + cap * B * 24) / args.steps,
                       "what": f"mgfwa_run_once(): create + init + {args.steps} generations + D2H, host-timed"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            e, s, what = cpu_reference_generation(w, 0, cores)
            line["cpu_baseline"] = {"value": e / s, "unit": "evals/s", "cores": cores, "kind": "reference",
                                    "sample": f"1 x {what} of the same workload, compiled reference, "
                                              f"data_parallel({cores}), {s:.1f} s"}
        except Exception as ex:  # the reference build travels in oracle/_ref
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if sharded:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

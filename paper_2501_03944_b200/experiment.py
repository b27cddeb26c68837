"""Experiment harness on the B200 engine — the GPU mode of the reference's
bench layer, mirroring
/root/reference/proj/include/mgfwa/bench.hpp and src/bench.cpp:

* ``ExperimentConfig`` / ``validate`` / ``normalized`` (bench.cpp:18-49),
  ``search_space_for`` (:70-76), ``objective_name`` (:83-88);
* ``run_experiment`` (:118-137): ``runs`` independent device-resident runs
  with seeds ``base_seed + r``;
* ``run_curve`` / ``best_at`` (:90-116), ``checkpoint_grid`` /
  ``default_checkpoints`` (:148-181), ``summarize`` (:183-205);
* ``write_trace_csv`` / ``write_summary_csv`` / ``format_double``
  (:207-235): the same CSV formats, doubles as ``%.17g``;
* ``compare`` / ``write_compare_report`` (:237-334).

Modes: the reference's ``serial`` (one population, one worker) and
``parallel`` (B batches over the data-parallel backend) both run on the GPU
engine here; the mode rules are kept (serial forces ``batches = 1``), the
worker count is meaningless on the device and is ignored.  ``compare`` thus
reports the B-batch over single-batch throughput ratio of the engine.
Objectives: ``net_id = 0`` is the sphere and ``net_id`` 1..12 the
reference's benchmark networks with ``weight_seed`` (``Net``, evaluated in
fp64 on the device), as in the reference; an explicit ``objective`` (any
device objective descriptor, e.g. ``MlpWeights()``) may be supplied instead.

CLI:  python -m paper_2501_03944_b200.experiment run --net 0 --dim 30 \\
          --runs 8 --max-evals 20000 --out DIR      (trace.csv, summary.csv)
      python -m paper_2501_03944_b200.experiment compare ... --out DIR
"""
from __future__ import annotations

import argparse
import dataclasses
import math
import os
import sys
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, TextIO

from .engine import NET_REGISTRY, MgfwaConfig, Net, Objective, RunRecord, SearchSpace, Sphere, run

SERIAL, PARALLEL = "serial", "parallel"


def mode_from_string(s: str) -> str:
    """mode_from_string, bench.cpp:12-16."""
    if s in (SERIAL, PARALLEL):
        return s
    raise ValueError("unknown mode: " + s)


@dataclass
class ExperimentConfig:
    """ExperimentConfig, bench.hpp:24-38 (+ an optional device objective)."""

    net_id: int = 0
    sphere_dim: int = 10
    mode: str = PARALLEL
    workers: int = 0
    algo: MgfwaConfig = field(default_factory=lambda: MgfwaConfig(max_evaluations=10000))
    lower: Optional[float] = None
    upper: Optional[float] = None
    runs: int = 8
    base_seed: int = 0
    weight_seed: int = 1
    out_dir: str = ""
    objective: Optional[Objective] = None  # overrides net_id when set
    dim: int = 0                           # search dimension for an analytic `objective`

    def validate(self) -> None:
        """ExperimentConfig::validate, bench.cpp:18-35 (same messages)."""
        if self.net_id < 0 or self.net_id > 12:
            raise ValueError("net id must be in 1..12")
        if self.net_id == 0 and self.sphere_dim == 0:
            raise ValueError("sphere dimension must be positive")
        if self.runs < 1:
            raise ValueError("runs must be >= 1")
        if self.workers < 0:
            raise ValueError("workers must be >= 0")
        if (self.lower is None) != (self.upper is None):
            raise ValueError("lower and upper bounds must be set together")
        if self.lower is not None and not (self.lower < self.upper):
            raise ValueError("bounds require lower < upper")
        self.algo.validate()


def normalized(config: ExperimentConfig) -> ExperimentConfig:
    """normalized, bench.cpp:37-46: serial forces one batch (and one worker)."""
    out = dataclasses.replace(config, algo=dataclasses.replace(config.algo))
    if out.mode == SERIAL:
        out.workers = 1
        out.algo.batches = 1
    elif out.workers == 0:
        out.workers = 1  # one device; the worker count does not apply
    return out


def _objective(config: ExperimentConfig) -> Objective:
    if config.objective is not None:
        return config.objective
    if config.net_id == 0:
        return Sphere()
    return Net(config.net_id, config.weight_seed)


def search_space_for(config: ExperimentConfig) -> SearchSpace:
    """search_space_for, bench.cpp:70-76 (uniform box)."""
    obj = _objective(config)
    if config.objective is not None:
        dim = obj.dim(config.dim)
        lo = config.lower if config.lower is not None else -1.0
        hi = config.upper if config.upper is not None else 1.0
    else:  # sphere(d) in [-10, 10], or net_spec(id).input_dim in [-5, 5]
        dim = config.sphere_dim if config.net_id == 0 else NET_REGISTRY[config.net_id][2]
        lo = config.lower if config.lower is not None else (-10.0 if config.net_id == 0 else -5.0)
        hi = config.upper if config.upper is not None else (10.0 if config.net_id == 0 else 5.0)
    if dim <= 0:
        raise ValueError("sphere dimension must be positive")
    return SearchSpace.box(dim, lo, hi)


def objective_name(config: ExperimentConfig) -> str:
    """objective_name, bench.cpp:83-88."""
    if config.objective is not None:
        return f"objective kind {config.objective.kind}"
    if config.net_id == 0:
        return f"sphere(d={config.sphere_dim})"
    return f"net {config.net_id}"


@dataclass
class WavePoint:
    evaluations: int = 0
    wall_ms: float = 0.0
    best: float = 0.0


@dataclass
class RunCurve:
    waves: List[WavePoint] = field(default_factory=list)


def run_curve(record: RunRecord) -> RunCurve:
    """run_curve, bench.cpp:90-107: best-so-far across batches per wave
    (evaluations and time of batch 0)."""
    curve = RunCurve()
    te, tb, tw = record.trace_evaluations, record.trace_best, record.trace_wall_ms
    if te.shape[0] == 0:
        return curve
    for w in range(te.shape[1]):
        best = float(tb[0, w])
        for b in range(1, tb.shape[0]):
            best = min(best, float(tb[b, w]))
        curve.waves.append(WavePoint(int(te[0, w]), float(tw[0, w]), best))
    return curve


def best_at(curve: RunCurve, t_ms: float) -> float:
    """best_at, bench.cpp:109-116."""
    best = curve.waves[0].best
    for p in curve.waves:
        if p.wall_ms > t_ms:
            break
        best = p.best
    return best


@dataclass
class ExperimentResult:
    config: ExperimentConfig
    records: List[RunRecord] = field(default_factory=list)
    curves: List[RunCurve] = field(default_factory=list)
    total_evaluations: int = 0
    total_wall_ms: float = 0.0


def run_experiment(config: ExperimentConfig, objective: Optional[Objective] = None,
                   space: Optional[SearchSpace] = None, device: int = 0) -> ExperimentResult:
    """run_experiment, bench.cpp:118-146: config.runs device runs, seeds
    base_seed + r."""
    config.validate()
    cfg = normalized(config)
    obj = objective if objective is not None else _objective(cfg)
    sp = space if space is not None else search_space_for(cfg)
    res = ExperimentResult(cfg)
    for r in range(cfg.runs):
        rec = run(cfg.algo, sp, obj, cfg.base_seed + r, device)
        res.total_evaluations += rec.evaluations_used
        res.curves.append(run_curve(rec))
        res.total_wall_ms += res.curves[-1].waves[-1].wall_ms
        res.records.append(rec)
    return res


def checkpoint_grid(t_max_ms: float, count: int = 16) -> List[float]:
    """checkpoint_grid, bench.cpp:148-166: log-spaced in (t_max/100, t_max]."""
    if not (t_max_ms > 0.0) or count == 0:
        raise ValueError("checkpoint_grid: needs positive span and count")
    t_min = t_max_ms / 100.0
    if count == 1:
        return [t_max_ms]
    ratio = t_max_ms / t_min
    grid = [t_min * math.pow(ratio, i / (count - 1)) for i in range(count)]
    grid[-1] = t_max_ms
    return grid


def default_checkpoints(result: ExperimentResult) -> List[float]:
    """default_checkpoints, bench.cpp:168-181."""
    t_max = result.config.algo.wall_clock_budget_ms
    if not (t_max > 0.0):
        t_max = math.inf
        for c in result.curves:
            t_max = min(t_max, c.waves[-1].wall_ms)
        if not (t_max > 0.0):
            t_max = 1.0
    return checkpoint_grid(t_max)


@dataclass
class SummaryRow:
    checkpoint_ms: float = 0.0
    mean_best: float = 0.0
    std_best: float = 0.0
    runs: int = 0


def summarize(result: ExperimentResult, checkpoints: Sequence[float]) -> List[SummaryRow]:
    """summarize, bench.cpp:183-205 (sample standard deviation)."""
    rows = []
    runs = len(result.curves)
    for t in checkpoints:
        mean = 0.0
        for c in result.curves:
            mean += best_at(c, t)
        mean /= runs
        var = 0.0
        for c in result.curves:
            dev = best_at(c, t) - mean
            var += dev * dev
        rows.append(SummaryRow(t, mean, math.sqrt(var / (runs - 1)) if runs > 1 else 0.0, runs))
    return rows


def format_double(v: float) -> str:
    """format_double, bench.cpp:207-211: printf("%.17g")."""
    return "%.17g" % v


def write_trace_csv(out: TextIO, result: ExperimentResult) -> None:
    """write_trace_csv, bench.cpp:213-225."""
    out.write("run_id,batch,evals,wall_ms,best_fitness\n")
    for r, rec in enumerate(result.records):
        for b in range(rec.trace_evaluations.shape[0]):
            for w in range(rec.trace_evaluations.shape[1]):
                out.write(f"{r},{b},{int(rec.trace_evaluations[b, w])},"
                          f"{format_double(float(rec.trace_wall_ms[b, w]))},"
                          f"{format_double(float(rec.trace_best[b, w]))}\n")


def write_summary_csv(out: TextIO, rows: Sequence[SummaryRow]) -> None:
    """write_summary_csv, bench.cpp:227-233."""
    out.write("checkpoint_ms,mean_best,std_best,runs\n")
    for row in rows:
        out.write(f"{format_double(row.checkpoint_ms)},{format_double(row.mean_best)},"
                  f"{format_double(row.std_best)},{row.runs}\n")


@dataclass
class ModeStats:
    evaluations: int = 0
    wall_ms: float = 0.0
    evals_per_second: float = 0.0


@dataclass
class Crossing:
    threshold: float = 0.0
    serial_reached: bool = False
    parallel_reached: bool = False
    serial_ms: float = 0.0
    parallel_ms: float = 0.0


@dataclass
class CompareReport:
    serial: ModeStats = field(default_factory=ModeStats)
    parallel: ModeStats = field(default_factory=ModeStats)
    speedup: float = 0.0
    crossings: List[Crossing] = field(default_factory=list)
    serial_curve: List[SummaryRow] = field(default_factory=list)
    parallel_curve: List[SummaryRow] = field(default_factory=list)


def compare(shared: ExperimentConfig, objective: Optional[Objective] = None,
            space: Optional[SearchSpace] = None, device: int = 0) -> CompareReport:
    """compare, bench.cpp:237-300: both modes, identical seeds; curves on a
    shared 64-point grid; first crossings of 50/90/99% of the improvement."""
    s_cfg = dataclasses.replace(shared, mode=SERIAL)
    p_cfg = dataclasses.replace(shared, mode=PARALLEL)
    serial = run_experiment(s_cfg, objective, space, device)
    parallel = run_experiment(p_cfg, objective, space, device)

    def stats(res: ExperimentResult) -> ModeStats:
        eps = res.total_evaluations / (res.total_wall_ms / 1e3) if res.total_wall_ms > 0.0 else 0.0
        return ModeStats(res.total_evaluations, res.total_wall_ms, eps)

    rep = CompareReport(serial=stats(serial), parallel=stats(parallel))
    rep.speedup = (rep.parallel.evals_per_second / rep.serial.evals_per_second
                   if rep.serial.evals_per_second > 0.0 else 0.0)
    t_max = shared.algo.wall_clock_budget_ms
    if not (t_max > 0.0):
        t_max = min(serial.curves[0].waves[-1].wall_ms, parallel.curves[0].waves[-1].wall_ms)
        for curves in (serial.curves, parallel.curves):
            for c in curves:
                t_max = min(t_max, c.waves[-1].wall_ms)
        if not (t_max > 0.0):
            t_max = 1.0
    grid = checkpoint_grid(t_max, 64)
    rep.serial_curve = summarize(serial, grid)
    rep.parallel_curve = summarize(parallel, grid)
    start = max(rep.serial_curve[0].mean_best, rep.parallel_curve[0].mean_best)
    floor = min(rep.serial_curve[-1].mean_best, rep.parallel_curve[-1].mean_best)
    for q in (0.5, 0.9, 0.99):
        cr = Crossing(threshold=start - q * (start - floor))
        for i, t in enumerate(grid):
            if not cr.serial_reached and rep.serial_curve[i].mean_best <= cr.threshold:
                cr.serial_reached, cr.serial_ms = True, t
            if not cr.parallel_reached and rep.parallel_curve[i].mean_best <= cr.threshold:
                cr.parallel_reached, cr.parallel_ms = True, t
        rep.crossings.append(cr)
    return rep


def write_compare_report(out: TextIO, rep: CompareReport) -> None:
    """write_compare_report, bench.cpp:310-332."""
    def mode_line(name, st):
        out.write(f"{name}: {st.evaluations} evaluations in {format_double(st.wall_ms)} ms "
                  f"({format_double(st.evals_per_second)} evals/s)\n")

    mode_line("serial  ", rep.serial)
    mode_line("parallel", rep.parallel)
    out.write(f"throughput ratio (parallel/serial): {format_double(rep.speedup)}\n")
    out.write("first crossings:\n")
    for cr in rep.crossings:
        out.write(f"  fitness <= {format_double(cr.threshold)}: serial ")
        out.write(f"{format_double(cr.serial_ms)} ms" if cr.serial_reached else "not reached")
        out.write(", parallel ")
        out.write(f"{format_double(cr.parallel_ms)} ms" if cr.parallel_reached else "not reached")
        out.write("\n")


# ------------------------------------------------------------------- CLI
def _config_from_args(a) -> ExperimentConfig:
    algo = MgfwaConfig(batches=a.batches, fireworks=a.fireworks, sparks_per_firework=a.sparks,
                       guides_per_firework=a.guides, boosts=[1.0, 2.0, 4.0, 8.0][: a.guides],
                       max_evaluations=a.max_evals, wall_clock_budget_ms=a.wall_ms)
    return ExperimentConfig(net_id=a.net, sphere_dim=a.dim, mode=a.mode, algo=algo, lower=a.lower,
                            upper=a.upper, runs=a.runs, base_seed=a.seed, out_dir=a.out or "")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2501_03944_b200.experiment")
    ap.add_argument("command", choices=["run", "compare"])
    ap.add_argument("--net", type=int, default=0)
    ap.add_argument("--dim", type=int, default=10)
    ap.add_argument("--mode", default=PARALLEL, type=mode_from_string)
    ap.add_argument("--batches", type=int, default=1)
    ap.add_argument("--fireworks", type=int, default=5)
    ap.add_argument("--sparks", type=int, default=30)
    ap.add_argument("--guides", type=int, default=3)
    ap.add_argument("--max-evals", type=int, default=20000)
    ap.add_argument("--wall-ms", type=float, default=0.0)
    ap.add_argument("--lower", type=float, default=None)
    ap.add_argument("--upper", type=float, default=None)
    ap.add_argument("--runs", type=int, default=8)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    a = ap.parse_args(argv)
    cfg = _config_from_args(a)
    try:
        if a.command == "run":
            res = run_experiment(cfg)
            if not cfg.out_dir:
                write_trace_csv(sys.stdout, res)
                return 0
            os.makedirs(cfg.out_dir, exist_ok=True)
            with open(os.path.join(cfg.out_dir, "trace.csv"), "w") as f:
                write_trace_csv(f, res)
            with open(os.path.join(cfg.out_dir, "summary.csv"), "w") as f:
                write_summary_csv(f, summarize(res, default_checkpoints(res)))
            print(f"{objective_name(res.config)}: {res.total_evaluations} evaluations in "
                  f"{format_double(res.total_wall_ms)} ms; wrote trace.csv and summary.csv")
        else:
            rep = compare(cfg)
            write_compare_report(sys.stdout, rep)
            if cfg.out_dir:
                os.makedirs(cfg.out_dir, exist_ok=True)
                for name, rows in (("compare_serial.csv", rep.serial_curve),
                                   ("compare_parallel.csv", rep.parallel_curve)):
                    with open(os.path.join(cfg.out_dir, name), "w") as f:
                        write_summary_csv(f, rows)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())


__all__ = ["ExperimentConfig", "ExperimentResult", "RunCurve", "WavePoint", "SummaryRow", "CompareReport",
           "Crossing", "ModeStats", "mode_from_string", "normalized", "search_space_for", "objective_name",
           "run_experiment", "run_curve", "best_at", "checkpoint_grid", "default_checkpoints", "summarize",
           "format_double", "write_trace_csv", "write_summary_csv", "compare", "write_compare_report"]

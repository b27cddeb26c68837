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

CLI (cli.cpp's mgfwa_bench: subcommands run / compare / nets, the same
flags, JSON config keys, messages and exit codes 0 / 2 / 3):
      python -m paper_2501_03944_b200.experiment run --sphere 30 --runs 8 \\
          --budget-evals 20000 --out DIR           (trace.csv, summary.csv)
      python -m paper_2501_03944_b200.experiment compare --net 5 ... --out DIR
      python -m paper_2501_03944_b200.experiment nets
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
    algo: MgfwaConfig = field(default_factory=MgfwaConfig)
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
# cli.cpp:22-380 (mgfwa_bench run / compare / nets) without CLI11: the same
# subcommands, flags, JSON config keys, messages and exit codes.
EXIT_OK, EXIT_INVALID_ARGS, EXIT_IO_FAILURE = 0, 2, 3  # cli.hpp:6-8

_JSON_KEYS = {"net", "sphere", "mode", "workers", "batches", "mu", "lambda", "guides", "sigma", "beta", "ca",
              "cr", "a0", "lower", "upper", "runs", "seed", "weight_seed", "budget_ms", "budget_evals", "out"}


def apply_json_config(path: str, cfg: ExperimentConfig) -> bool:
    """apply_json_config, cli.cpp:22-78; returns whether an objective was set."""
    import json

    try:
        with open(path) as f:
            doc = json.load(f)
    except OSError:
        raise ValueError("cannot read config file: " + path)
    selected = False
    for key, value in doc.items():
        if key not in _JSON_KEYS:
            raise ValueError("unknown config key: " + key)
        selected |= _apply(cfg, key, value)
    return selected


def _apply(cfg: ExperimentConfig, key: str, value) -> bool:
    a = cfg.algo
    if key == "net":
        cfg.net_id = int(value)
        return True
    if key == "sphere":
        cfg.sphere_dim, cfg.net_id = int(value), 0
        return True
    setters = {
        "mode": lambda v: setattr(cfg, "mode", mode_from_string(v)),
        "workers": lambda v: setattr(cfg, "workers", int(v)),
        "batches": lambda v: setattr(a, "batches", int(v)),
        "mu": lambda v: setattr(a, "fireworks", int(v)),
        "lambda": lambda v: setattr(a, "sparks_per_firework", int(v)),
        "guides": lambda v: setattr(a, "guides_per_firework", int(v)),
        "sigma": lambda v: setattr(a, "guide_fraction", float(v)),
        "beta": lambda v: setattr(a, "boosts", [float(x) for x in v]),
        "ca": lambda v: setattr(a, "amp_amplify", float(v)),
        "cr": lambda v: setattr(a, "amp_reduce", float(v)),
        "a0": lambda v: setattr(a, "initial_amplitude", float(v)),
        "lower": lambda v: setattr(cfg, "lower", float(v)),
        "upper": lambda v: setattr(cfg, "upper", float(v)),
        "runs": lambda v: setattr(cfg, "runs", int(v)),
        "seed": lambda v: setattr(cfg, "base_seed", int(v)),
        "weight_seed": lambda v: setattr(cfg, "weight_seed", int(v)),
        "budget_ms": lambda v: setattr(a, "wall_clock_budget_ms", float(v)),
        "budget_evals": lambda v: setattr(a, "max_evaluations", int(v)),
        "out": lambda v: setattr(cfg, "out_dir", str(v)),
    }
    setters[key](value)
    return False


def algorithm_params_match(x: ExperimentConfig, y: ExperimentConfig) -> bool:
    """algorithm_params_match, bench.cpp:48-63."""
    ax, ay = x.algo, y.algo
    return (x.net_id == y.net_id and x.sphere_dim == y.sphere_dim and ax.fireworks == ay.fireworks
            and ax.sparks_per_firework == ay.sparks_per_firework
            and ax.guides_per_firework == ay.guides_per_firework and ax.guide_fraction == ay.guide_fraction
            and list(ax.boosts) == list(ay.boosts) and ax.amp_amplify == ay.amp_amplify
            and ax.amp_reduce == ay.amp_reduce and ax.initial_amplitude == ay.initial_amplitude
            and ax.max_evaluations == ay.max_evaluations and ax.wall_clock_budget_ms == ay.wall_clock_budget_ms
            and x.lower == y.lower and x.upper == y.upper and x.runs == y.runs and x.base_seed == y.base_seed
            and x.weight_seed == y.weight_seed)


_FLAG_KEYS = [("net", "net"), ("sphere", "sphere"), ("mode", "mode"), ("workers", "workers"),
              ("batches", "batches"), ("mu", "mu"), ("lambda_", "lambda"), ("guides", "guides"),
              ("sigma", "sigma"), ("beta", "beta"), ("ca", "ca"), ("cr", "cr"), ("a0", "a0"),
              ("lower", "lower"), ("upper", "upper"), ("runs", "runs"), ("seed", "seed"),
              ("weight_seed", "weight_seed"), ("budget_ms", "budget_ms"), ("budget_evals", "budget_evals"),
              ("out", "out")]


def resolve_config(args) -> tuple:
    """resolve_config, cli.cpp:131-191: defaults, then the JSON file, then the
    flags actually given; default boost ladder 1, 2, 4, ... when only the
    guide count changed."""
    cfg = ExperimentConfig(algo=MgfwaConfig())
    selected = False
    if args.config:
        selected = apply_json_config(args.config, cfg)
    for attr, key in _FLAG_KEYS:
        v = getattr(args, attr, None)
        if v is None:
            continue
        if key == "beta":
            v = [float(x) for x in v.split(",")]
        selected |= _apply(cfg, key, v)
        if key == "guides" and cfg.algo.guides_per_firework == 0:
            cfg.algo.boosts = []
    a = cfg.algo
    if a.guides_per_firework > 0 and len(a.boosts) != a.guides_per_firework and args.beta is None:
        a.boosts = [2.0 ** i for i in range(a.guides_per_firework)]
    return cfg, selected


def do_run(cfg: ExperimentConfig) -> int:
    """do_run, cli.cpp:209-245."""
    if not cfg.out_dir:
        raise ValueError("run requires --out DIR")
    try:
        os.makedirs(cfg.out_dir, exist_ok=True)
    except OSError:
        raise IOError("cannot create " + cfg.out_dir)
    res = run_experiment(cfg)
    trace_path = os.path.join(cfg.out_dir, "trace.csv")
    summary_path = os.path.join(cfg.out_dir, "summary.csv")
    with open(trace_path, "w") as f:
        write_trace_csv(f, res)
    with open(summary_path, "w") as f:
        write_summary_csv(f, summarize(res, default_checkpoints(res)))
    best = min(c.waves[-1].best for c in res.curves)
    print(f"{objective_name(res.config)}, {res.config.mode} mode, {len(res.records)} runs: best fitness "
          f"{format_double(best)}, {res.total_evaluations} evaluations total\n"
          f"wrote {trace_path} and {summary_path}")
    return EXIT_OK


def do_compare(shared: ExperimentConfig) -> int:
    """do_compare, cli.cpp:247-284 (curves as wall_ms,best_fitness)."""
    if not shared.out_dir:
        raise ValueError("compare requires --out DIR")
    try:
        os.makedirs(shared.out_dir, exist_ok=True)
    except OSError:
        raise IOError("cannot create " + shared.out_dir)
    rep = compare(shared)
    paths = []
    for name, rows in (("compare_serial.csv", rep.serial_curve), ("compare_parallel.csv", rep.parallel_curve)):
        path = os.path.join(shared.out_dir, name)
        with open(path, "w") as f:
            f.write("wall_ms,best_fitness\n")
            for row in rows:
                f.write(f"{format_double(row.checkpoint_ms)},{format_double(row.mean_best)}\n")
        paths.append(path)
    write_compare_report(sys.stdout, rep)
    print(f"wrote {paths[0]} and {paths[1]}")
    return EXIT_OK


def do_nets() -> int:
    """do_nets, cli.cpp:286-297."""
    from .engine import net_param_count

    print("id,scale,activation,input_dim,hidden_dim,output_dim,hidden_layers,params,reported_params")
    for nid, (scale, act, d, h, lh, rep) in NET_REGISTRY.items():
        print(f"{nid},{scale},{act},{d},{h},1,{lh},{net_param_count(nid)},{rep}")
    return EXIT_OK


def _parser():
    ap = argparse.ArgumentParser(prog="python -m paper_2501_03944_b200.experiment",
                                 description="Batched multi-guiding-spark fireworks optimizer benchmark (B200)")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p, with_mode):
        p.add_argument("--config")
        g = p.add_mutually_exclusive_group()
        g.add_argument("--net", type=int, choices=range(1, 13), metavar="{1..12}")
        g.add_argument("--sphere", type=int)
        if with_mode:
            p.add_argument("--mode")
        p.add_argument("--workers", type=int)
        p.add_argument("--batches", "-B", type=int)
        p.add_argument("--mu", type=int)
        p.add_argument("--lambda", dest="lambda_", type=int)
        p.add_argument("--guides", "-M", type=int)
        p.add_argument("--sigma", type=float)
        p.add_argument("--beta")
        p.add_argument("--ca", type=float)
        p.add_argument("--cr", type=float)
        p.add_argument("--a0", type=float)
        p.add_argument("--lower", type=float)
        p.add_argument("--upper", type=float)
        p.add_argument("--runs", type=int)
        p.add_argument("--seed", type=int)
        p.add_argument("--weight-seed", dest="weight_seed", type=int)
        p.add_argument("--budget-ms", dest="budget_ms", type=float)
        p.add_argument("--budget-evals", dest="budget_evals", type=int)
        p.add_argument("--out")

    common(sub.add_parser("run", help="optimize one objective and write trace/summary CSVs"), True)
    c = sub.add_parser("compare", help="run serial and parallel modes on shared parameters and seeds")
    common(c, False)
    c.add_argument("--serial-config", dest="serial_config")
    c.add_argument("--parallel-config", dest="parallel_config")
    sub.add_parser("nets", help="list the 12 benchmark networks")
    return ap


def main(argv=None) -> int:
    """cli_main, cli.cpp:301-380: exit codes 0 / 2 (invalid arguments) /
    3 (I/O failure)."""
    try:
        args = _parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_INVALID_ARGS
    try:
        if args.command == "nets":
            return do_nets()
        cfg, selected = resolve_config(args)
        if not selected:
            raise ValueError("choose an objective: --net <1..12> or --sphere <D>")
        if args.command == "run":
            cfg.validate()
            return do_run(cfg)
        if args.serial_config or args.parallel_config:
            s_cfg = dataclasses.replace(cfg, algo=dataclasses.replace(cfg.algo))
            p_cfg = dataclasses.replace(cfg, algo=dataclasses.replace(cfg.algo))
            if args.serial_config:
                apply_json_config(args.serial_config, s_cfg)
            if args.parallel_config:
                apply_json_config(args.parallel_config, p_cfg)
            if not algorithm_params_match(s_cfg, p_cfg):
                raise ValueError("serial and parallel configs disagree on algorithm parameters")
            cfg = p_cfg
        cfg.validate()
        return do_compare(cfg)
    except (IOError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO_FAILURE
    except (ValueError, KeyError, TypeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INVALID_ARGS


if __name__ == "__main__":
    sys.exit(main())


__all__ = ["ExperimentConfig", "ExperimentResult", "RunCurve", "WavePoint", "SummaryRow", "CompareReport",
           "Crossing", "ModeStats", "mode_from_string", "normalized", "search_space_for", "objective_name",
           "run_experiment", "run_curve", "best_at", "checkpoint_grid", "default_checkpoints", "summarize",
           "format_double", "write_trace_csv", "write_summary_csv", "compare", "write_compare_report",
           "apply_json_config", "algorithm_params_match", "resolve_config", "main"]

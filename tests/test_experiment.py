"""Experiment harness (paper_2501_03944_b200.experiment), the GPU mode of
the reference's bench layer.  Mirrors the
reference's tests/test_bench.cpp cases: validation messages, mode rules,
checkpoint grid, trace CSV format and determinism, summary statistics
against an independent recomputation from the CSV, serial/parallel paths.
"""
import io
import math

import numpy as np
import pytest

import paper_2501_03944_b200 as P
from paper_2501_03944_b200 import experiment as E


def _record(evals, best, wall):
    """A RunRecord with the given [batch][wave] traces (CPU-only tests)."""
    evals, best, wall = (np.atleast_2d(np.asarray(a)) for a in (evals, best, wall))
    return P.RunRecord(config=P.MgfwaConfig(max_evaluations=1), space=P.SearchSpace.box(1, -1, 1), seed=0,
                       trace_evaluations=evals.astype(np.uint64), trace_best=best.astype(float),
                       trace_wall_ms=wall.astype(float), best_position=np.zeros((evals.shape[0], 1)),
                       best_fitness=best[:, -1].astype(float), evaluations_used=int(evals[0, -1]),
                       iterations=evals.shape[1] - 1, losers_reinitialized=0, nan_evaluations=0)


# ------------------------------------------------------------------ CPU
def test_validation_messages():
    cases = [(dict(net_id=13), "net id must be in 1..12"), (dict(net_id=-1), "net id must be in 1..12"),
             (dict(sphere_dim=0), "sphere dimension must be positive"), (dict(runs=0), "runs must be >= 1"),
             (dict(workers=-1), "workers must be >= 0"),
             (dict(lower=-1.0), "lower and upper bounds must be set together"),
             (dict(lower=1.0, upper=1.0), "bounds require lower < upper")]
    for kw, msg in cases:
        with pytest.raises(ValueError, match=msg):
            E.ExperimentConfig(**kw).validate()
    with pytest.raises(ValueError, match="at least one budget"):
        E.ExperimentConfig(algo=P.MgfwaConfig()).validate()
    with pytest.raises(ValueError, match="unknown mode: fast"):
        E.mode_from_string("fast")


def test_mode_rules_and_space():
    cfg = E.ExperimentConfig(mode=E.SERIAL, algo=P.MgfwaConfig(batches=4, max_evaluations=100), workers=8)
    n = E.normalized(cfg)
    assert n.algo.batches == 1 and n.workers == 1 and cfg.algo.batches == 4  # input untouched
    assert E.normalized(E.ExperimentConfig(algo=P.MgfwaConfig(batches=4, max_evaluations=9))).algo.batches == 4
    sp = E.search_space_for(E.ExperimentConfig(sphere_dim=7))
    assert sp.dim() == 7 and sp.lower[0] == -10.0 and sp.upper[0] == 10.0
    assert E.objective_name(E.ExperimentConfig(sphere_dim=7)) == "sphere(d=7)"
    sp = E.search_space_for(E.ExperimentConfig(net_id=3))  # net_spec(3).input_dim, [-5, 5]
    assert sp.dim() == 20 and sp.lower[0] == -5.0 and sp.upper[0] == 5.0
    assert E.objective_name(E.ExperimentConfig(net_id=3)) == "net 3"


def test_checkpoint_grid_matches_reference_formula():
    g = E.checkpoint_grid(250.0, 16)
    assert len(g) == 16 and g[-1] == 250.0 and g[0] == pytest.approx(2.5)
    for i in range(15):  # log-spaced: constant ratio (bench.cpp:148-166)
        assert g[i + 1] / g[i] == pytest.approx(100.0 ** (1 / 15))
    assert E.checkpoint_grid(3.0, 1) == [3.0]
    with pytest.raises(ValueError, match="checkpoint_grid: needs positive span and count"):
        E.checkpoint_grid(0.0)
    with pytest.raises(ValueError):
        E.checkpoint_grid(1.0, 0)


def test_format_double_round_trips():
    for v in (0.1, 1.0 / 3.0, 1e-320, 123456789.123456789, -2.5e300):
        s = E.format_double(v)
        assert float(s) == v and s == "%.17g" % v


def test_curves_summary_and_csv_on_synthetic_records():
    r0 = _record([[5, 10, 15], [5, 10, 15]], [[9.0, 4.0, 4.0], [8.0, 8.0, 1.0]], [[1.0, 2.0, 3.0], [1.0, 2.0, 3.0]])
    r1 = _record([[5, 10, 15], [5, 10, 15]], [[7.0, 6.0, 2.0], [9.0, 5.0, 5.0]], [[0.5, 2.5, 4.0], [0.5, 2.5, 4.0]])
    res = E.ExperimentResult(E.ExperimentConfig(algo=P.MgfwaConfig(max_evaluations=15)), [r0, r1])
    res.curves = [E.run_curve(r) for r in (r0, r1)]
    assert [w.best for w in res.curves[0].waves] == [8.0, 4.0, 1.0]  # min over batches per wave
    assert E.best_at(res.curves[1], 0.1) == 7.0 and E.best_at(res.curves[1], 3.0) == 5.0
    rows = E.summarize(res, [1.0, 2.5, 10.0])
    assert rows[0].mean_best == pytest.approx((8.0 + 7.0) / 2)
    assert rows[1].mean_best == pytest.approx((4.0 + 5.0) / 2)
    assert rows[2].std_best == pytest.approx(math.sqrt(((1 - 1.5) ** 2 + (2 - 1.5) ** 2) / 1))
    out = io.StringIO()
    E.write_trace_csv(out, res)
    lines = out.getvalue().splitlines()
    assert lines[0] == "run_id,batch,evals,wall_ms,best_fitness"
    assert len(lines) == 1 + 2 * 2 * 3 and lines[1] == "0,0,5,1,9"
    out = io.StringIO()
    E.write_summary_csv(out, rows)
    assert out.getvalue().splitlines()[0] == "checkpoint_ms,mean_best,std_best,runs"


# ------------------------------------------------------------------ GPU
def _sphere_config(**kw):
    algo = P.MgfwaConfig(batches=2, fireworks=4, sparks_per_firework=12, guides_per_firework=2,
                         boosts=[1.0, 2.0], guide_fraction=0.25, max_evaluations=8 + 30 * 2 * 4 * 14)
    base = dict(sphere_dim=6, runs=3, algo=algo)
    base.update(kw)
    return E.ExperimentConfig(**base)


def _strip_wall(csv):
    return ["".join(f for i, f in enumerate(l.split(",")) if i != 3) for l in csv.splitlines()]


def _parse_trace(csv):
    runs = {}
    for line in csv.splitlines()[1:]:
        r, b, ev, wall, best = line.split(",")
        runs.setdefault(int(r), {}).setdefault(int(ev), []).append((float(wall), float(best)))
    return runs


@pytest.mark.gpu
def test_initialization_only_trace():
    cfg = _sphere_config(runs=1)
    cfg.algo.max_evaluations = cfg.algo.batches * cfg.algo.fireworks
    res = E.run_experiment(cfg)
    assert res.records[0].trace_evaluations.shape[1] == 1
    out = io.StringIO()
    E.write_trace_csv(out, res)
    assert len(out.getvalue().splitlines()) == 1 + cfg.algo.batches


@pytest.mark.gpu
def test_trace_csv_deterministic_apart_from_wall_clock():
    a, b = io.StringIO(), io.StringIO()
    E.write_trace_csv(a, E.run_experiment(_sphere_config()))
    E.write_trace_csv(b, E.run_experiment(_sphere_config()))
    assert _strip_wall(a.getvalue()) == _strip_wall(b.getvalue())
    assert a.getvalue().splitlines()[0] == "run_id,batch,evals,wall_ms,best_fitness"


@pytest.mark.gpu
def test_summary_matches_recomputation_from_csv():
    res = E.run_experiment(_sphere_config(runs=8))
    cps = E.default_checkpoints(res)
    rows = E.summarize(res, cps)
    out = io.StringIO()
    E.write_trace_csv(out, res)
    runs = _parse_trace(out.getvalue())
    assert len(runs) == 8 and len(rows) == len(cps)
    for t, row in zip(cps, rows):
        bests = []
        for waves in runs.values():
            ordered = sorted(waves.items())
            best = min(p[1] for p in ordered[0][1])
            for _, pts in ordered:
                if pts[0][0] <= t:  # batch 0's time stamp (run_curve)
                    best = min(p[1] for p in pts)
            bests.append(best)
        mean = sum(bests) / len(bests)
        std = math.sqrt(sum((x - mean) ** 2 for x in bests) / (len(bests) - 1))
        assert row.runs == 8
        assert row.mean_best == pytest.approx(mean, rel=1e-9)
        assert row.std_best == pytest.approx(std, rel=1e-9, abs=1e-300)


@pytest.mark.gpu
def test_serial_and_parallel_walk_the_same_path():
    cfg = _sphere_config()
    cfg.algo.batches = 1
    s = E.run_experiment(E.ExperimentConfig(**{**cfg.__dict__, "mode": E.SERIAL}))
    p = E.run_experiment(E.ExperimentConfig(**{**cfg.__dict__, "mode": E.PARALLEL, "workers": 2}))
    for cs, cp in zip(s.curves, p.curves):
        assert [w.evaluations for w in cs.waves] == [w.evaluations for w in cp.waves]
        assert [w.best for w in cs.waves] == [w.best for w in cp.waves]


@pytest.mark.gpu
def test_compare_report_and_cli(tmp_path):
    rep = E.compare(_sphere_config(runs=2))
    assert rep.serial.evaluations > 0 and rep.parallel.evaluations > rep.serial.evaluations
    assert len(rep.serial_curve) == 64 and len(rep.crossings) == 3
    out = io.StringIO()
    E.write_compare_report(out, rep)
    assert out.getvalue().startswith("serial  : ")
    rc = E.main(["run", "--sphere", "5", "--runs", "2", "--budget-evals", "600", "--out", str(tmp_path)])
    assert rc == 0
    assert (tmp_path / "trace.csv").read_text().startswith("run_id,batch,evals,wall_ms,best_fitness\n")
    assert (tmp_path / "summary.csv").read_text().startswith("checkpoint_ms,mean_best,std_best,runs\n")
    rc = E.main(["compare", "--net", "1", "-B", "2", "--lambda", "12", "--guides", "2", "--runs", "2",
                 "--budget-evals", "2000", "--out", str(tmp_path / "cmp")])
    assert rc == 0
    assert (tmp_path / "cmp" / "compare_serial.csv").read_text().startswith("wall_ms,best_fitness\n")


def test_cli_config_resolution_and_errors(tmp_path, capsys):
    import json

    conf = tmp_path / "c.json"
    conf.write_text(json.dumps({"sphere": 12, "batches": 3, "guides": 4, "budget_evals": 1000, "seed": 9}))
    args = E._parser().parse_args(["run", "--config", str(conf), "--mu", "7"])
    cfg, selected = E.resolve_config(args)
    assert selected and cfg.sphere_dim == 12 and cfg.algo.batches == 3 and cfg.algo.fireworks == 7
    assert cfg.algo.boosts == [1.0, 2.0, 4.0, 8.0] and cfg.base_seed == 9  # default ladder (cli.cpp:180-189)
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"sphere": 3, "colour": 1}))
    assert E.main(["run", "--config", str(bad), "--out", str(tmp_path)]) == E.EXIT_INVALID_ARGS
    assert "unknown config key: colour" in capsys.readouterr().err
    assert E.main(["run", "--budget-evals", "10", "--out", str(tmp_path)]) == E.EXIT_INVALID_ARGS
    assert "choose an objective: --net <1..12> or --sphere <D>" in capsys.readouterr().err
    assert E.main(["run", "--sphere", "4", "--budget-evals", "10"]) == E.EXIT_INVALID_ARGS
    assert "run requires --out DIR" in capsys.readouterr().err
    assert E.main(["run", "--net", "13"]) == E.EXIT_INVALID_ARGS
    assert E.main(["run", "--config", str(tmp_path / "missing.json")]) == E.EXIT_INVALID_ARGS
    assert "cannot read config file" in capsys.readouterr().err
    s = tmp_path / "s.json"
    s.write_text(json.dumps({"mu": 4}))
    assert E.main(["compare", "--sphere", "3", "--budget-evals", "100", "--serial-config", str(s),
                   "--out", str(tmp_path)]) == E.EXIT_INVALID_ARGS
    assert "serial and parallel configs disagree on algorithm parameters" in capsys.readouterr().err


def test_cli_nets_listing(capsys):
    assert E.main(["nets"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "id,scale,activation,input_dim,hidden_dim,output_dim,hidden_layers,params,reported_params"
    assert lines[1] == "1,small,relu,10,16,1,2,465,465"
    assert lines[10] == "10,large,gelu,1000,512,1,11,3139585,3137585"  # nets 10-12: nearest realizable

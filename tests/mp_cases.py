"""Solves shared by the two-process test (tests/test_gpu_multiprocess.py):
run in each rank of the torch.distributed job and, for comparison, in one
process with two local shards. Results are JSON-exact (floats by repr)."""
from paper_2601_17196_b200 import pot

CASES = ("aspot_f64", "feasible_f64", "tuned_f64", "aspot_f32_points")


def _setup(name):
    if name == "aspot_f32_points":
        inst = pot.config_instance(3, n=2048)
        cfg = pot.SolverConfig(epsilon=2e-2, log_every=10 ** 9, max_iterations=200, materialize_plan=False,
                               collect_iter_log=True)
        return inst, pot.SolverKind.Aspot, cfg
    inst = pot.config_instance(1, n=600)
    kind = {"aspot_f64": pot.SolverKind.Aspot, "feasible_f64": pot.SolverKind.FeasibleSinkhorn,
            "tuned_f64": pot.SolverKind.TunedSinkhorn}[name]
    cfg = pot.SolverConfig(epsilon=1e-2, tuning_exponent_p=2.0, log_every=10 ** 9, materialize_plan=False,
                           collect_iter_log=(kind == pot.SolverKind.Aspot))
    return inst, kind, cfg


def run_case(name, ctx):
    inst, kind, cfg = _setup(name)
    g = pot.solve(inst, kind, cfg, ctx=ctx, iter_log_cap=100000) if kind == pot.SolverKind.Aspot else \
        pot.solve(inst, kind, cfg, ctx=ctx)
    out = {"status": int(g.status), "iterations": int(g.iterations), "cost": float(g.cost),
           "gap": float(g.feasibility_gap), "phi": float(g.phi), "final_error": float(g.final_error),
           "row_slack_sum": float(g.plan.row_slack.sum()), "col_slack_sum": float(g.plan.col_slack.sum())}
    if g.iter_log is not None:
        out["log"] = g.iter_log.tolist()
    return out


def oracle_case(name):
    from oracle import binding
    inst, kind, cfg = _setup(name)
    return binding.solve(int(kind), inst.r, inst.c, inst.s, C=inst.C, epsilon=cfg.epsilon,
                         p=cfg.tuning_exponent_p, log_every=10 ** 9, want_plan=False)

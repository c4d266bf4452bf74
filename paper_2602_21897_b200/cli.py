"""`python -m paper_2602_21897_b200.cli run|sweep|dag` -- the reference's
`taskweave` subcommands (tools/main.cpp:92-119) for the CG workload on the
CUDA backend.  Config precedence: --config file < TASKWEAVE_* env < flags.
Exit codes: 0 ok, 1 ConfigError, 2 ContractViolation (main.cpp:139-151)."""
from __future__ import annotations

import argparse
import sys

from . import scenario as S
from ._native import ConfigError, ContractViolation


def assemble(argv: list) -> tuple:
    ap = argparse.ArgumentParser(prog="taskweave-b200")
    ap.add_argument("command", choices=["run", "sweep", "dag", "keys"])
    ap.add_argument("--config")
    for k in S.config_keys():
        ap.add_argument("--" + k.replace("_", "-"), dest=k)
    ap.add_argument("--iteration", type=int, default=0, help="dag: iteration to export")
    a = ap.parse_args(argv)
    c = S.ScenarioConfig()
    if a.config:
        S.apply_config_file(c, a.config)
    S.apply_env(c)
    for k in S.config_keys():
        v = getattr(a, k)
        if v is not None:
            S.apply_key(c, k, v)
    c.validate()
    return a, c


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    try:
        a, c = assemble(argv)
        if a.command == "keys":
            print("\n".join(S.config_keys()))
        elif a.command in ("run", "sweep"):
            tiles = c.tiles if a.command == "sweep" else c.tiles[:1]
            points = [S.run_point(c, t) for t in tiles]
            sys.stdout.write(S.metrics_to_csv(points))
        else:
            from . import hpccg as H
            A = H.gen_stencil_matrix(c.nx, c.ny, c.nz)
            tiles = H.make_tile_plan(A, c.tiles[0])
            edges = H.task_dag_edges(A.n, tiles, a.iteration + 1)
            tag = f":{a.iteration}:"
            print("digraph deps {")
            for u, v in edges:
                if tag in u and tag in v:
                    print(f'  "{u}" -> "{v}";')
            print("}")
        return 0
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 1
    except ContractViolation as e:
        print(f"contract violation: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

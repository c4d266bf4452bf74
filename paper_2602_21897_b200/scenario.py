"""Scenario harness for the CUDA backend: the reference's ScenarioConfig keys
and its 11-column metrics CSV.

Mirrors proj/include/taskweave/{config,scenario}.hpp and
proj/src/{config,scenario}.cpp for the CG workload:

* the same key set, parsed the same way (flat key=value files with '#'
  comments, TASKWEAVE_<KEY> environment variables, command-line flags; flags
  override env, env overrides file -- config.cpp:153-210, main.cpp:32-42);
  ``backend`` gains the value ``cuda``, the only one that runs here;
* the same CSV header and row format (scenario.cpp:177-247, %.17g doubles);
* the same warm-up rule (scenario.cpp:262-263) and scenario ids
  (config.cpp:246-260).

``iter_time`` is device-timed seconds per iteration (CUDA events at each
iteration end, tw_cg_iteration_times) rather than virtual cost units.  The
per-worker usage columns describe the one device "worker": busy = summed
iteration time, blocked / suspended / idle = 0.  ``tasks_executed`` counts
kernel launches (one per repetition when the tasks variant's automatic
dispatch picks the persistent dispatcher, > 8 tiles), ``events_polled`` the
completions the task-aware poller saw.
"""
from __future__ import annotations

import io
import os
from dataclasses import dataclass, field

import numpy as np

from . import hpccg as H
from ._native import ConfigError

VARIANTS = ("monolithic", "tasks")
BACKENDS = ("host", "device-blocking", "device-ta", "cuda")
MODES = ("single-rt", "multi-rt-uncoordinated", "multi-rt-unified")
CLOCKS = ("virtual", "real")
WORKLOADS = ("cg", "pipeline")


@dataclass
class ScenarioConfig:
    """ScenarioConfig (config.hpp:26-52) with backend=cuda available."""
    scenario_id: str = ""
    workload: str = "cg"
    variant: str = "tasks"
    tiles: list = field(default_factory=lambda: [16])
    backend: str = "cuda"
    mode: str = "single-rt"
    workers: int = 4
    clock: str = "real"
    repetitions: int = 1
    seed: int = 7
    poll_period: float = 0.5
    pool_count: int = 4
    pool_threads: int = 8
    stream_pool: int = 4
    iterations: int = 50
    warmup: int = 10
    nx: int = 32
    ny: int = 32
    nz: int = 32
    use_graph: bool = False  # B200 extension (not a reference key)

    def validate(self) -> None:
        """ScenarioConfig::validate (config.cpp:213-244) + the device backend."""
        if not self.tiles:
            raise ConfigError("tiles sweep list is empty")
        if any(t < 1 for t in self.tiles):
            raise ConfigError("tile count must be >= 1")
        if self.workers < 1:
            raise ConfigError("workers must be >= 1")
        if self.repetitions < 1:
            raise ConfigError("repetitions must be >= 1")
        if self.iterations < 1:
            raise ConfigError("iterations must be >= 1")
        if self.warmup < 0:
            raise ConfigError("warmup must be >= 0")
        if self.poll_period <= 0:
            raise ConfigError("poll_period must be > 0")
        if self.pool_count < 1 or self.pool_threads < 1:
            raise ConfigError("pool_count and pool_threads must be >= 1")
        if self.stream_pool < 1:
            raise ConfigError("stream_pool must be >= 1")
        if self.nx < 1 or self.ny < 1 or self.nz < 1:
            raise ConfigError("stencil dims must be >= 1")
        if self.variant == "monolithic" and any(t != 1 for t in self.tiles):
            raise ConfigError("monolithic variant requires tiles=1")
        if self.workload != "cg":
            raise ConfigError("the B200 build implements the cg workload only")
        if self.backend != "cuda":
            raise ConfigError(f"backend '{self.backend}' runs on the reference's simulated "
                              "device; the B200 build provides backend=cuda")

    def id_for(self, tile: int) -> str:
        """ScenarioConfig::id_for (config.cpp:246-260)."""
        if self.scenario_id:
            return f"{self.scenario_id}-t{tile}"
        return (f"{self.workload}-{self.variant}-{self.backend}-{self.mode}"
                f"-w{self.workers}-t{tile}")


def _int(v: str, key: str) -> int:
    try:
        if v.strip() != v or v == "":
            raise ValueError
        return int(v, 10)
    except ValueError:
        raise ConfigError(f"key '{key}': expected an integer, got '{v}'") from None


def _float(v: str, key: str) -> float:
    try:
        return float(v)
    except ValueError:
        raise ConfigError(f"key '{key}': expected a number, got '{v}'") from None


def _choice(v: str, choices, key: str) -> str:
    if v not in choices:
        raise ConfigError(f"key '{key}': unknown value '{v}' (expected one of "
                          f"{', '.join(choices)})")
    return v


def _int_list(v: str, key: str) -> list:
    out = [_int(x, key) for x in v.split(",")] if v else []
    if not out:
        raise ConfigError(f"key '{key}': empty list")
    return out


_SETTERS = {
    "scenario_id": lambda c, k, v: setattr(c, "scenario_id", v),
    "workload": lambda c, k, v: setattr(c, "workload", _choice(v, WORKLOADS, k)),
    "variant": lambda c, k, v: setattr(c, "variant", _choice(v, VARIANTS, k)),
    "tiles": lambda c, k, v: setattr(c, "tiles", _int_list(v, k)),
    "backend": lambda c, k, v: setattr(c, "backend", _choice(v, BACKENDS, k)),
    "mode": lambda c, k, v: setattr(c, "mode", _choice(v, MODES, k)),
    "workers": lambda c, k, v: setattr(c, "workers", _int(v, k)),
    "clock": lambda c, k, v: setattr(c, "clock", _choice(v, CLOCKS, k)),
    "repetitions": lambda c, k, v: setattr(c, "repetitions", _int(v, k)),
    "seed": lambda c, k, v: setattr(c, "seed", _int(v, k)),
    "poll_period": lambda c, k, v: setattr(c, "poll_period", _float(v, k)),
    "pool_count": lambda c, k, v: setattr(c, "pool_count", _int(v, k)),
    "pool_threads": lambda c, k, v: setattr(c, "pool_threads", _int(v, k)),
    "stream_pool": lambda c, k, v: setattr(c, "stream_pool", _int(v, k)),
    "iterations": lambda c, k, v: setattr(c, "iterations", _int(v, k)),
    "warmup": lambda c, k, v: setattr(c, "warmup", _int(v, k)),
    "nx": lambda c, k, v: setattr(c, "nx", _int(v, k)),
    "ny": lambda c, k, v: setattr(c, "ny", _int(v, k)),
    "nz": lambda c, k, v: setattr(c, "nz", _int(v, k)),
    "use_graph": lambda c, k, v: setattr(c, "use_graph", bool(_int(v, k))),
}
# pipeline keys exist in the reference's key set; accepted, unused here
for _k in ("pl_batch", "pl_context", "pl_channels", "pl_out_channels", "pl_b_gran", "pl_t_gran"):
    _SETTERS[_k] = lambda c, k, v: _int(v, k)


def config_keys() -> list:
    return sorted(_SETTERS)


def apply_key(c: ScenarioConfig, key: str, value: str) -> None:
    """apply_key (config.cpp:153-158)."""
    if key not in _SETTERS:
        raise ConfigError(f"unknown config key '{key}'")
    _SETTERS[key](c, key, value)


def apply_config_stream(c: ScenarioConfig, text: str, name: str) -> None:
    """Flat key=value lines, '#' comments, name:line diagnostics (config.cpp:167-193)."""
    for lineno, line in enumerate(text.splitlines(), 1):
        s = line.lstrip(" \t")
        if not s or s[0] == "#":
            continue
        if "=" not in line:
            raise ConfigError(f"{name}:{lineno}: expected key=value")
        key, value = line.split("=", 1)
        key = key.strip(" \t")
        value = value.strip(" \t\r")
        try:
            apply_key(c, key, value)
        except ConfigError as e:
            raise ConfigError(f"{name}:{lineno}: {e}") from None


def apply_config_file(c: ScenarioConfig, path: str) -> None:
    try:
        text = open(path).read()
    except OSError:
        raise ConfigError(f"cannot open config file '{path}'") from None
    apply_config_stream(c, text, path)


def apply_env(c: ScenarioConfig, env=None) -> None:
    """TASKWEAVE_<KEY> overrides (config.cpp:202-210)."""
    env = os.environ if env is None else env
    for key in config_keys():
        var = "TASKWEAVE_" + key.upper()
        if var in env:
            apply_key(c, key, env[var])


# ------------------------------------------------------------------ CSV

HEADER = ("scenario,repetition,iteration,warmup,iter_time,busy,blocked,suspended,idle,"
          "tasks_executed,events_polled")


def metrics_csv_header() -> str:
    return HEADER


def _g(v: float) -> str:
    return "%.17g" % v


@dataclass
class MetricsRow:
    """MetricsRow (scenario.hpp:16-27)."""
    scenario: str
    repetition: int
    iteration: int
    warmup: bool
    iter_time: float
    busy: list
    blocked: list
    suspended: list
    idle: list
    tasks_executed: int
    events_polled: int


def to_csv_row(r: MetricsRow) -> str:
    """to_csv_row (scenario.cpp:182-196)."""
    j = lambda vs: ";".join(_g(v) for v in vs)  # noqa: E731
    return ",".join([r.scenario, str(r.repetition), str(r.iteration), "1" if r.warmup else "0",
                     _g(r.iter_time), j(r.busy), j(r.blocked), j(r.suspended), j(r.idle),
                     str(r.tasks_executed), str(r.events_polled)])


def parse_metrics_csv(text: str) -> list:
    """parse_metrics_csv (scenario.cpp:198-247)."""
    out, saw = [], False
    for lineno, line in enumerate(io.StringIO(text).read().splitlines(), 1):
        line = line.rstrip("\r")
        if not line:
            continue
        if not saw:
            if line != HEADER:
                raise ConfigError(f"metrics csv line {lineno}: unexpected header '{line}'")
            saw = True
            continue
        f = line.split(",")
        try:
            if len(f) != 11:
                raise ConfigError(f"expected 11 comma-separated fields, got {len(f)}")
            if f[3] not in ("0", "1"):
                raise ConfigError("warmup flag must be 0 or 1")
            sp = lambda s: [float(x) for x in s.split(";")] if s else []  # noqa: E731
            out.append(MetricsRow(f[0], int(f[1]), int(f[2]), f[3] == "1", float(f[4]),
                                  sp(f[5]), sp(f[6]), sp(f[7]), sp(f[8]), int(f[9]),
                                  int(f[10])))
        except (ValueError, ConfigError) as e:
            raise ConfigError(f"metrics csv line {lineno}: {e}") from None
    if not saw:
        raise ConfigError("metrics csv: missing header")
    return out


@dataclass
class PointResult:
    """PointResult (scenario.hpp:35-46)."""
    tile: int
    rows: list
    residual_history: np.ndarray
    steady_iter_time: float


def run_point(c: ScenarioConfig, tile: int, rt: H.Runtime | None = None) -> PointResult:
    """run_point (scenario.cpp:249-291) on the CUDA backend."""
    c.validate()
    rt = rt or H.default_runtime()
    A = H.gen_stencil_matrix(c.nx, c.ny, c.nz, rt=rt)
    b = H.rhs_splitmix(rt, A.n, c.seed)  # SplitMix64(seed), scenario.cpp:91-95
    variant = H.N.TW_CG_MONOLITHIC if c.variant == "monolithic" else H.N.TW_CG_TASKS
    opt = H.CgOptions(tiles=tile, stream_pool_capacity=c.stream_pool, iteration_marks=True,
                      use_graph=c.use_graph, auto_dispatch=True)
    rows, hist = [], None
    steady, allv = [], []
    for rep in range(c.repetitions):
        S = H.CgSolver(rt, A, c.iterations, opt, variant=variant)
        try:
            S.set_rhs(b)
            S.iterate(c.iterations)
            times = S.iteration_times(c.iterations)
            hist = S.history(c.iterations)
            kernels, _ = S.launches_per_iteration()
            launches = kernels * c.iterations if kernels else 1  # persistent: one launch
            polled = c.iterations
        finally:
            S.close()
        busy = float(np.sum(times))
        for i, t in enumerate(times):
            warm = (c.repetitions > 1 and rep == 0) or i < c.warmup
            rows.append(MetricsRow(c.id_for(tile), rep, i, warm, float(t), [busy], [0.0],
                                   [0.0], [0.0], launches, polled))
            allv.append(float(t))
            if not warm:
                steady.append(float(t))
    st = float(np.mean(steady)) if steady else (float(np.mean(allv)) if allv else 0.0)
    return PointResult(tile, rows, hist, st)


def run_sweep(c: ScenarioConfig, rt: H.Runtime | None = None) -> list:
    c.validate()
    return [run_point(c, t, rt) for t in c.tiles]


def metrics_to_csv(points: list) -> str:
    lines = [HEADER] + [to_csv_row(r) for p in points for r in p.rows]
    return "\n".join(lines) + "\n"

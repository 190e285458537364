"""TrainConfig and DensifySchedule and the
per-iteration event schedule of the train op.

TrainConfig serialises to JSON losslessly and rejects unknown keys;
`--set key=value` overrides follow the CLI contract."""
from __future__ import annotations

import dataclasses
import json
from dataclasses import dataclass, field

from . import types as T


class ConfigError(ValueError):
    """Validation error (the reference CLI's exit code 1)."""


@dataclass
class DensifySchedule:
    warmup: int = 600
    interval: int = 100
    end: int = 14900
    opacity_reset_interval: int = 3000
    grad_threshold: float = 2e-4
    prune_opacity: float = 0.05
    morton_interval: int = 5000
    sh_ramp: int = 1000

    def validate(self, total_iterations: int) -> None:
        for f in dataclasses.fields(self):
            if not getattr(self, f.name) > 0:
                raise ConfigError(f"densify.{f.name} must be positive")
        if self.end > total_iterations:
            raise ConfigError("densify.end exceeds total_iterations")


@dataclass
class TrainConfig:
    total_iterations: int = 30000
    bound_mode: int = T.BOUND_RECT_OPACITY
    cull_mode: int = T.CULL_EXACT
    sort_mode: str = "two_stage"
    backward_mode: int = T.BACKWARD_PER_PIXEL
    optimizer_mode: int = T.ADAM_FUSED
    morton: bool = True
    aa_mode: str = "off"          # off | filter3d_original | filter3d_clip | full
    kappa3d: float = 0.2          # 3D filter variance
    rate_interval: int = 100      # sampling-rate recompute interval
    truncation: str = "classic"   # classic | response
    sigma_cut: float = 3.33        # response truncation cutoff (sigmas)
    dynamic_4d: bool = False
    batch_size: int = 1
    seed: int = 0
    dataset: str = ""
    output_dir: str = ""
    checkpoint_interval: int = 5000
    densify: DensifySchedule = field(default_factory=DensifySchedule)

    # ---- validation / (de)serialisation ----
    def validate(self) -> "TrainConfig":
        if self.total_iterations < 0 or self.batch_size < 1 or self.checkpoint_interval < 1:
            raise ConfigError("total_iterations >= 0, batch_size >= 1, checkpoint_interval >= 1 required")
        if self.sort_mode not in ("two_stage", "combined"):
            raise ConfigError(f"sort_mode {self.sort_mode!r}")
        if self.aa_mode not in T.AA_MODES:
            raise ConfigError(f"aa_mode {self.aa_mode!r}: one of {sorted(T.AA_MODES)} (SPEC.md:675)")
        if not self.kappa3d > 0 or self.rate_interval < 1:
            raise ConfigError("kappa3d > 0 and rate_interval >= 1 required")
        if self.truncation not in ("classic", "response") or not self.sigma_cut > 0:
            raise ConfigError("truncation: classic | response, sigma_cut > 0 (SPEC.md:319)")
        if self.dynamic_4d:
            raise ConfigError("dynamic_4d: the 4D extension is not on the B200 path")
        if self.backward_mode not in (T.BACKWARD_PER_PIXEL, T.BACKWARD_PER_GAUSSIAN):
            raise ConfigError(f"backward_mode {self.backward_mode}")
        if self.optimizer_mode not in range(5):
            raise ConfigError(f"optimizer_mode {self.optimizer_mode}")
        self.densify.validate(self.total_iterations)
        return self

    def to_dict(self) -> dict:
        return dataclasses.asdict(self)

    @classmethod
    def from_dict(cls, d: dict) -> "TrainConfig":
        d = dict(d)
        known = {f.name for f in dataclasses.fields(cls)}
        bad = set(d) - known
        if bad:
            raise ConfigError(f"unknown config keys: {sorted(bad)}")
        dens = d.pop("densify", {})
        dknown = {f.name for f in dataclasses.fields(DensifySchedule)}
        if set(dens) - dknown:
            raise ConfigError(f"unknown densify keys: {sorted(set(dens) - dknown)}")
        return cls(**d, densify=DensifySchedule(**dens))

    def dumps(self) -> str:
        return json.dumps(self.to_dict(), indent=1, sort_keys=True)

    @classmethod
    def loads(cls, s: str) -> "TrainConfig":
        return cls.from_dict(json.loads(s))

    def save(self, path) -> None:
        with open(path, "w") as f:
            f.write(self.dumps())

    @classmethod
    def load(cls, path) -> "TrainConfig":
        with open(path) as f:
            return cls.loads(f.read())

    def override(self, assignments) -> "TrainConfig":
        """Apply `key=value` strings (dotted keys reach densify.*); values parsed as JSON when possible."""
        d = self.to_dict()
        for a in assignments:
            if "=" not in a:
                raise ConfigError(f"--set expects key=value, got {a!r}")
            k, v = a.split("=", 1)
            try:
                val = json.loads(v)
            except json.JSONDecodeError:
                val = v
            tgt, parts = d, k.split(".")
            for p in parts[:-1]:
                if p not in tgt or not isinstance(tgt[p], dict):
                    raise ConfigError(f"unknown config key {k!r}")
                tgt = tgt[p]
            if parts[-1] not in tgt:
                raise ConfigError(f"unknown config key {k!r}")
            tgt[parts[-1]] = val
        return TrainConfig.from_dict(d)


@dataclass(frozen=True)
class Events:
    sh_degree: int
    densify: bool
    opacity_reset: bool
    morton: bool
    checkpoint: bool


def events(it: int, cfg: TrainConfig) -> Events:
    """What fires after the optimizer step of iteration `it` (1-based)."""
    s = cfg.densify
    active = it <= s.end
    return Events(
        sh_degree=min(3, (it - 1) // s.sh_ramp) if it > 0 else 0,
        densify=active and it >= s.warmup and it % s.interval == 0,
        opacity_reset=active and it % s.opacity_reset_interval == 0,
        morton=cfg.morton and active and it % s.morton_interval == 0,
        checkpoint=it % cfg.checkpoint_interval == 0,
    )

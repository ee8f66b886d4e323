"""Static parameters, batch shapes and step results (the reference's env/core.py:24-94).

``StaticParams`` validates exactly as ``env/core.py:35-48`` and additionally rejects
what the CUDA kernels do not support (grids above 16x16 or 128 interior cells, view
sizes above 9, episodes longer than 65535 steps) with the same ``ConfigError``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

from . import _lib
from .errors import ConfigError


@dataclass(frozen=True)
class StaticParams:
    height: int = 13
    width: int = 13
    max_episode_steps: int = 250
    agent_view_size: int = 5
    wall_budget: int = 60
    see_through_walls: bool = True

    def validate(self) -> "StaticParams":
        if self.height < 3 or self.width < 3:
            raise ConfigError(f"grid must be at least 3x3, got {self.height}x{self.width}")
        if self.agent_view_size < 3 or self.agent_view_size % 2 == 0:
            raise ConfigError(f"agent_view_size must be odd and >= 3, got {self.agent_view_size}")
        if self.max_episode_steps < 1:
            raise ConfigError(f"max_episode_steps must be >= 1, got {self.max_episode_steps}")
        top = self.n_interior - 2
        if not 0 <= self.wall_budget <= top:
            raise ConfigError(f"wall_budget must be in [0, {top}] for a {self.height}x{self.width} grid, "
                              f"got {self.wall_budget}")
        if self.height > 16 or self.width > 16 or self.n_interior > 128:
            raise ConfigError(f"grid {self.height}x{self.width} exceeds the 16x16 / 128-cell kernel limit")
        if self.agent_view_size > 9:
            raise ConfigError(f"agent_view_size {self.agent_view_size} > 9 is not supported")
        if self.max_episode_steps > 65535:
            raise ConfigError(f"max_episode_steps {self.max_episode_steps} > 65535 is not supported")
        return self

    @property
    def n_interior(self) -> int:
        return (self.height - 2) * (self.width - 2)

    def c_struct(self) -> _lib.AmzParams:
        return _lib.AmzParams(self.height, self.width, self.max_episode_steps, self.agent_view_size,
                              self.wall_budget, int(bool(self.see_through_walls)))


def as_params(p) -> StaticParams:
    """Accept ours or the reference's StaticParams (same field names)."""
    if isinstance(p, StaticParams):
        return p
    return StaticParams(p.height, p.width, p.max_episode_steps, p.agent_view_size, p.wall_budget,
                        bool(p.see_through_walls))


@dataclass
class StepResult:
    """reset/step return value (env/core.py:55-69).  Arrays are torch CUDA tensors."""

    observation: Any
    state: Any
    reward: Any
    done: Any
    info: dict = field(default_factory=dict)
    extras: dict = field(default_factory=dict)


@dataclass(frozen=True)
class BatchShape:
    """population x evaluations x instances; inner two flattened (env/core.py:72-94)."""

    n_agents: int = 1
    n_evals: int = 1
    n_envs: int = 1

    def __post_init__(self):
        if min(self.n_agents, self.n_evals, self.n_envs) < 1:
            raise ConfigError(f"batch dimensions must all be >= 1, got {self}")

    @property
    def flat_size(self) -> int:
        return self.n_evals * self.n_envs

    @property
    def total(self) -> int:
        return self.n_agents * self.flat_size

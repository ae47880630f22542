"""IntegrationResult -- the return type of phsp_average (integrate.py:23-33).

The reference's plain-MC / Gauss-Kronrod / VEGAS integrators are outside this
package's scope (not on the north_star path); the phase-space
integral is phsp_average / phsp_integrate.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class IntegrationResult:
    value: float
    error: float
    iterations: int = 1
    chi2_per_dof: float = 0.0
    calls_used: int = 0

    @property
    def converged(self) -> bool:
        return math.isfinite(self.value) and math.isfinite(self.error)

"""Wrench -> rotor-thrust allocation (EXTENSION: not in the reference).

The reference commands (f, M) directly onto the rigid body and has no rotor
model.  BASELINE.json configs 0 and 4 ask for X-quad and
hexarotor allocation, so this module defines it:
rotor i at arm_length * (cos a_i, sin a_i, 0) in the body frame (z-up),
spin s_i = +-1, thrust T_i >= 0 along +b3, drag torque s_i * kappa * T_i
about +b3.  The wrench is A T with column i = (1, y_i, -x_i, s_i kappa);
the kernel evaluates T = clip(A^+ w, 0, rotor_max) with A^+ = A^T (A A^T)^-1
computed here in float64.  Constants are builder-chosen.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class Airframe:
    name: str
    angles_deg: tuple
    spins: tuple
    arm_length: float = 0.2      # m, hub to rotor
    kappa: float = 0.05          # m, drag-torque / thrust ratio
    rotor_max: float = 10.0      # N per rotor

    @property
    def n_rotors(self) -> int:
        return len(self.angles_deg)

    def matrix(self) -> np.ndarray:
        a = np.deg2rad(np.asarray(self.angles_deg, dtype=np.float64))
        x, y = self.arm_length * np.cos(a), self.arm_length * np.sin(a)
        s = np.asarray(self.spins, dtype=np.float64)
        return np.stack([np.ones_like(x), y, -x, s * self.kappa])

    def pinv(self) -> np.ndarray:
        a = self.matrix()
        return a.T @ np.linalg.inv(a @ a.T)

    def native(self) -> N.fs_airframe:
        f = N.fs_airframe()
        f.n_rotors = self.n_rotors
        f.rotor_max = self.rotor_max
        pinv = np.zeros((N.FS_MAX_ROTORS, 4))
        pinv[:self.n_rotors] = self.pinv()
        alloc = np.zeros((4, N.FS_MAX_ROTORS))
        alloc[:, :self.n_rotors] = self.matrix()
        f.pinv[:] = [float(x) for x in pinv.reshape(-1)]
        f.alloc[:] = [float(x) for x in alloc.reshape(-1)]
        return f


QUAD_X = Airframe("quad_x", (45.0, 135.0, 225.0, 315.0), (1, -1, 1, -1),
                  arm_length=0.2, kappa=0.05, rotor_max=10.0)
HEXAROTOR = Airframe("hex", (0.0, 60.0, 120.0, 180.0, 240.0, 300.0), (1, -1, 1, -1, 1, -1),
                     arm_length=0.2, kappa=0.05, rotor_max=7.0)


def native_pair(first: Airframe | None, second: Airframe | None = None):
    """(fs_airframe * 2) for the kernel: vehicles with global id < split use
    `first`, the others `second` (defaults to `first`)."""
    arr = (N.fs_airframe * 2)()
    if first is None:
        return None
    arr[0] = first.native()
    arr[1] = (second or first).native()
    return arr

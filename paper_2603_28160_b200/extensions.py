"""Extended kinematics: the BASELINE.json features the reference lacks.

The reference models a face mill with circular inserts, per-tooth radial /
axial run-out, straight-line feed and one pass. The
benchmark configurations additionally name ball-end tools, helix lag, a
tool-axis runout with a phase, lead tilt, radial vibration, per-flute edge
noise and raster passes. This module pins their definition;
with every field at its default the sweep runs the reference kinematics
bit-exactly, and ``force_extended=True`` with all-zero extensions runs the
extended formulation, which the tests show is bit-identical on the reference
goldens as well.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ConfigError


@dataclass(frozen=True)
class Extensions:
    """Definitions (tool frame of tooth K = the reference's edge->tool frame):

    profile: "insert" — reference circular-insert arc at radius D/2
        (tool_geometry.py:101-175); "ball" — the flute is the meridian
        arc of a sphere of radius R about (0, 0, R): polar angle kappa in
        [0, kappa_max], kappa_max = min(pi/2, acos((R-a_p)/R) + |tilt|),
        points uniform in kappa, placed at the axis (no D/2).
    helix_angle_rad (beta): a point at edge height h lags the tip by
        psi = h * tan(beta) / r_ref (r_ref = D/2 for insert, R for ball,
        or helix_ref_radius_mm); tool-frame (x, y) rotated by -psi.
    runout_offset_mm (rho), runout_phase_rad (lambda): tool-axis offset,
        a rigid translation (rho cos a_K, rho sin a_K) of tooth K's tool
        frame, a_K = lambda + 2 pi (K-1)/Z.
    tilt_rad (tau): lead tilt, rotation about the workpiece X axis applied
        after the spindle rotation: y' = cos(tau) y - sin(tau) z,
        z' = sin(tau) y + cos(tau) z, re-levelled so the lowest point the
        rotating tool can reach sits at z0.
    vib_amplitude_mm, vib_frequency_hz, vib_phase_rad: radial tool
        vibration along X, x0(t) += A sin(2 pi f t + phase).
    noise_sigma_mm, noise_corr_mm, noise_seed: per-flute edge-radius
        perturbation delta (Gaussian-smoothed white noise from
        numpy default_rng(seed), kernel std corr/(2 ds), rescaled to sigma)
        applied along the profile normal.
    passes, stepover_mm: raster of unidirectional (+Y) passes, pass k at
        x0 + k * stepover, merged by elementwise min (HeightField.merge_min).
    """

    profile: str = "insert"
    helix_angle_rad: float = 0.0
    helix_ref_radius_mm: float | None = None
    runout_offset_mm: float = 0.0
    runout_phase_rad: float = 0.0
    tilt_rad: float = 0.0
    vib_amplitude_mm: float = 0.0
    vib_frequency_hz: float = 0.0
    vib_phase_rad: float = 0.0
    noise_sigma_mm: float = 0.0
    noise_corr_mm: float = 0.0
    noise_seed: int = 0
    passes: int = 1
    stepover_mm: float = 0.0
    force_extended: bool = False

    def __post_init__(self) -> None:
        if self.profile not in ("insert", "ball"):
            raise ConfigError(f"profile must be 'insert' or 'ball', got {self.profile!r}")
        if not (0.0 <= abs(self.helix_angle_rad) < math.pi / 2):
            raise ConfigError(f"helix angle must satisfy |beta| < pi/2, got {self.helix_angle_rad}")
        if self.helix_ref_radius_mm is not None and self.helix_ref_radius_mm <= 0:
            raise ConfigError("helix_ref_radius_mm must be > 0")
        if abs(self.tilt_rad) >= math.pi / 2:
            raise ConfigError(f"tilt must satisfy |tau| < pi/2, got {self.tilt_rad}")
        if self.passes < 1:
            raise ConfigError(f"passes must be >= 1, got {self.passes}")
        if self.noise_sigma_mm < 0 or self.noise_corr_mm < 0:
            raise ConfigError("noise sigma and correlation length must be >= 0")
        if self.vib_amplitude_mm != 0.0 and self.vib_frequency_hz < 0:
            raise ConfigError("vibration frequency must be >= 0")

    @property
    def kinematic(self) -> bool:
        """True when the extended formulation is needed."""
        return bool(self.force_extended or self.profile != "insert" or self.helix_angle_rad != 0.0
                    or self.runout_offset_mm != 0.0 or self.tilt_rad != 0.0
                    or self.vib_amplitude_mm != 0.0 or self.noise_sigma_mm != 0.0)

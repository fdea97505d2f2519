"""Non-default PG discretisation modes (R/discretisation.py:164-224,279-286).

Off the production path (the drivers always use the anisotropic "xy" mode).
"""


def _todo(name):
    raise NotImplementedError(f"{name}: non-default discretisation mode not built yet "
                              "(SURVEY.md §8f item 3)")


def pg_isotropic_diffusivity(psi, fs, quad, cfg, mode="mixed_mass"):
    _todo("pg_isotropic_diffusivity")


def residual_estimate(psi, fs, quad, cfg, mode="mixed_mass"):
    _todo("residual_estimate")


def residual_alternatives(psi, fs, quad, cfg, mode):
    _todo("residual_alternatives")

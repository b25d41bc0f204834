"""Test-side re-export of the shared seeded input generators (no method arithmetic)."""
from paper_2301_01179_b200.inputs import (Problem, config_c1, config_c2, config_c3, config_c4,  # noqa: F401
                                          config_c5, surface_sources, uniform_rings)

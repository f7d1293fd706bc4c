"""Collapsed Gauss-Jacobi rules on the reference simplices (reference ``quadrature.py:30-66``),
re-exported under the reference's module name for drop-in imports; host-side setup only
(ErrorFunctional, operator checks)."""

from .modal import tet_rule, triangle_rule

__all__ = ["tet_rule", "triangle_rule"]

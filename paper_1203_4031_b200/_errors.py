"""Exception types shared by the drivers (mirrors _driver.py:20-21, reduced.py:15-16)."""


class SingularMatrixError(Exception):
    """Exactly singular pivot or inner-solver breakdown (maps to info -2)."""


class ReducedSolverError(Exception):
    """Iteration failure in the reduced eigensolver (maps to info -3)."""

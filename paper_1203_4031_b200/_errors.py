"""Exception types shared by the drivers (mirrors _driver.py:20-21, reduced.py:15-16)."""


class SingularMatrixError(ArithmeticError):
    """Exactly singular pivot or inner-solver breakdown (maps to info -2).

    An ArithmeticError, so that feastlib's own run_rci (which catches its own
    SingularMatrixError and ArithmeticError, _driver.py:55-57,88-89) maps it to
    info -2 when B200DenseOps / B200BandOps are plugged into the reference."""


class ReducedSolverError(Exception):
    """Iteration failure in the reduced eigensolver (maps to info -3)."""

"""Numeric mode selection (drop-in for pkg/src/nnjit/options.py:9-27).

The two reference fields keep their names, defaults and ``ValueError``
behaviour.  Each accepts one extra value:

* ``activation_mode="exact"`` evaluates tanh/sigmoid like the reference
  interpreter (float64 transcendental, rounded once to float32,
  pkg/src/nnjit/interpreter.py:102-112) instead of an approximation.
* ``softmax_exp="exact"`` does the same for softmax
  (pkg/src/nnjit/interpreter.py:115-118).

``"rational"``/``"fast"``/``"precise"`` are evaluated on the device with the
reference's operation order and no FMA contraction, so each element matches
the numpy models in pkg/src/nnjit/codegen/approx.py:72-128 bit for bit.
"""

from dataclasses import dataclass

ACTIVATION_MODES = ("rational", "fast", "exact")
SOFTMAX_EXP_MODES = ("fast", "precise", "exact")


@dataclass(frozen=True)
class ApproximationOptions:
    activation_mode: str = "rational"
    softmax_exp: str = "fast"

    def __post_init__(self):
        if self.activation_mode not in ACTIVATION_MODES:
            raise ValueError(f"activation_mode must be one of {ACTIVATION_MODES},"
                             f" got {self.activation_mode!r}")
        if self.softmax_exp not in SOFTMAX_EXP_MODES:
            raise ValueError(f"softmax_exp must be one of {SOFTMAX_EXP_MODES},"
                             f" got {self.softmax_exp!r}")


#: Interpreter-grade transcendentals everywhere: the mode the FP32 parity gate
#: (rtol 1e-4 / atol 1e-5 against the oracle) is run in.
EXACT = ApproximationOptions(activation_mode="exact", softmax_exp="exact")

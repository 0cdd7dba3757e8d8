"""B200-native LLG step (arXiv:1501.07293 reference `mmsim`): the per-step demag convolution,
local terms and explicit-Euler update as sm_100a kernels behind a C-ABI (include/mmb.h,
libmmb.so), with a Python mirror of the reference's SimulationBase interface."""
from .problems import (FieldSchedule, Grid, MaterialParams, ProblemSpec, ScheduleStage,  # noqa: F401
                       standard_problem_3_benchmark, standard_problem_4)
from .simulation import (Backend, Precision, RunOptions, Simulation, TrajectoryRecord,  # noqa: F401
                         backend_from_string, make_simulation, precision_from_string,
                         random_unit_field)
from .validate import ValidationReport, run_validation  # noqa: F401

"""paper_1811_01566_b200 -- B200-native B-mode reconstruction hot path.

Drop-in for the hot path of echopipe (the reference restatement of WaveFlow,
arXiv 1811.01566): Delay-and-Sum for STA and plane-wave imaging, analytic-
signal envelope detection and log compression, executed by hand-written
sm_100a CUDA kernels in ``_lib/libbmode200.so`` (C ABI: include/bmode200.h).
Public names mirror echopipe/__init__.py:9-64 for the path.
"""

from .beamform import (INTERPOLATION_MODES, DasPlan, active_aperture, das_beamform,
                       das_beamform_oracle)
from . import engine, parallel, qus
from .engine import BmodeEngine
from .environment import (DatasetSource, Environment, Phantom, SimulatorSource,
                          default_pw_angles, next_observation, open_dataset, open_simulator,
                          simulate_rf,
                          simulate_rf_device, wire_phantom)
from .formats import WfrfReader, read_wfrf, write_pgm, write_wfrf
from .errors import (AllZeroInput, AxisTooShort, DimensionMismatch, EchopipeError,
                     EmptyCoefficients, FormatError, InvalidMetadata, NativeError,
                     NonPositiveRange, OperatorFailed, WindowTooLarge, WrongStage)
from .pipeline import (OPERATOR_REGISTRY, BenchmarkResult, OperatorKind, PipelineGraph,
                       StageTiming, benchmark, bmode_chain, build_graph, execute,
                       register_gpu_operators, register_operator)
from .qus import (DenseLayer, DenseModel, HkParamsMap, MomentMaps, dense_forward,
                  estimate_hk_map, load_model, save_model, sliding_moments)
from .sigproc import FirSpec, analytic_signal, dynamic_adjustment, envelope, fir_filter
from .types import (AcquisitionContext, ApodizationSpec, BmodeImage, ImageGrid, PwScheme,
                    RfFrame, StaScheme, centered_rx_map, default_grid, validate_pair)

__version__ = "0.1.0"

"""B200-native FEPLL restoration loop (arXiv:1710.08124) — drop-in for the
reference package's ``restore`` entry point and degradation-operator
interface.  See DESIGN.md for the kernel map and INTEGRATION.md for the
C ABI."""

__version__ = "0.1.0"

from .errors import DataError, DeviceError, FepllError, NumericalError
from .gmm import (Eigenbasis, FlatTailComponent, GmmModel, component_from_eigen,
                  eigen_from_covariance, flatten_component, score_flat_cost, wiener_flat_cost)
from .model_io import model_read, model_write, tree_read, tree_write
from .operators import (CgConfig, DegradationOperator, SolveInfo, convolution_operator,
                        decimate_operator, gain_operator, gaussian_kernel, identity_operator,
                        mask_operator, radial_gain_map)
from .patches import SampleGrid, axis_anchors, jitter_rng, jittered_grid, regular_grid
from .solver import (HostPipeline, IterationStats, RestorationConfig, Restorer, SolverStats,
                     beta_schedule, cached_restorer, clear_plan_cache, restore, restore_batch)
from .tree import GmmTree, TreeNode
from .tree_build import auto_level_sizes, balanced_cluster, build_tree, pairwise_symmetric_kl

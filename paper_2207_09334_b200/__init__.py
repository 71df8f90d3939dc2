"""B200-native mass-spring relaxation loop (Cronos, arXiv 2207.09334).

Drop-in for the hot path of the reference ``springsim`` package: scene
construction (model/lattice), ``Engine`` (step/forces/state/commands) and
``simulate``, with the per-step work in hand-written sm_100a CUDA kernels
behind a C ABI (``include/springsim_b200.h``).  See DESIGN.md.
"""

from .engine import (
    EULER,
    EXEC_MODES,
    INTEGRATORS,
    PARALLEL,
    PARALLEL_DET,
    PRECISIONS,
    RK4,
    SERIAL,
    VERLET,
    DivergenceError,
    Engine,
    EngineState,
    RunResult,
    contact_force,
    energy_breakdown,
    simulate,
    spring_force,
    total_force,
)
from .lattice import (
    PITCH,
    beam_lattice,
    block_cells,
    block_scene,
    block_springs,
    crawler_scene,
    excite,
    multi_material_cube,
    voxel_arrays,
    voxel_box,
)
from .model import (
    ActuationGroup,
    ArrayScene,
    ContactPlane,
    Mass,
    Material,
    Scene,
    Spring,
    Violation,
    actuated_rest_length,
    contact_floor,
    scene_arrays,
    validate_scene,
)
from .traces import TraceSeries
from .batch import per_instance, replicate
from ._lib import pinned_copy, pinned_empty
from .sceneio import SceneFormatError, load_scene, parse_scene, render_scene, save_scene

__version__ = "0.1.0"

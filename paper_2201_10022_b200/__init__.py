"""B200-native ABD (arXiv 2201.10022) implicit Newton step.

Drop-in for the hot path of the reference `stiffbody` package: the
scene/step API below keeps the reference names and signatures
(`stiffbody/__init__.py:1-130`) and runs on hand-written fp64 sm_100a
kernels through the C-ABI in include/abd_b200.h.  There is no CPU
fallback: compute calls raise if libabd_b200.so or the GPU is missing.
Setup-time types (meshes, masses, shapes) are host code.
"""
from .aabb import Aabb, aabb_of, aabb_overlap
from .body import (
    BodyCoords,
    BodyMaterial,
    BodyState,
    GeneralizedMass,
    external_generalized_force,
    jacobian,
    mass_matrix,
    ortho_energy,
    ortho_error,
    ortho_gradient,
    ortho_hessian,
    project_psd,
    torque_point_forces,
    world_position,
    world_positions,
)
from .ccd import CcdQuery, accd_toi, accd_toi_batch, step_filter
from .constraints import (
    Reduction,
    ReparamMap,
    VirtualTet,
    build_constrained_system,
    constrain_linear,
    make_axis_tet,
    make_free_tet,
    phi,
    reparam_map,
)
from .contact import (
    BarrierDomainError,
    CandidateSet,
    CollisionBody,
    ContactPair,
    FrictionData,
    PairBlocks,
    barrier,
    barrier_d1,
    barrier_d2,
    broad_phase,
    candidate_min_distance_sq,
    contact_energy,
    contact_gradient_hessian,
    friction_energy,
    friction_gradient_hessian,
    friction_precompute,
    world_positions_all,
)
from .distance import (
    DistanceResult,
    EERegion,
    PTRegion,
    edge_edge_closest,
    edge_edge_distance_sq,
    ee_mollifier,
    ee_mollifier_grad_hess,
    pair_distance_gradients,
    point_triangle_closest,
    point_triangle_distance_sq,
)
from .intersect import intersecting_body_pairs, triangles_intersect, triangles_intersect_batch
from .mesh import SurfaceMesh, build_edges
from .scene import FrameStats, SceneConfig, SceneState, audit_intersections, load_scene, read_obj, run, write_obj_frame
from .shapes import box_mesh, icosphere_mesh, prism_mesh, torus_mesh, wedge_mesh
from .solver import (
    IncrementalPotentialState,
    SimState,
    StepFailure,
    StepParams,
    StepStats,
    SystemModel,
    advance_step,
    assemble,
    compute_q_tilde,
    global_min_distance,
    ip_value,
    line_search,
    solve_newton_system,
)
from .sparse import BlockCholesky, BlockJacobiPCG, BlockSparseMatrix, FactorizationError

__all__ = [n for n in dir() if not n.startswith("_")]
__version__ = "0.1.0"

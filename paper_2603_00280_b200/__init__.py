"""B200-native macrofacet volumetric path tracing (arXiv 2603.00280).

Drop-in for the hot path of the reference `macrofacet` package: the medium /
phase-function / integrator entry points and the scene description keep the
reference's names and signatures, and run as hand-written sm_100a CUDA
kernels behind the C ABI in include/macrofacet_b200.h.  No CPU fallback."""

__version__ = "0.1.0"

from . import gp
from .core import (Frame, build_frame, direction_to_spherical, dot, erf, erfc, gauss_cdf,
                   gauss_pdf, normalize, reflect, spherical_to_direction)
from .curves import (beckmann_ndf, density, fresnel_conductor, gdf_pdf, generalized_lambda,
                     generalized_lambda_dir, generalized_ndf, generalized_ndf_dir, ggx_ndf,
                     ndf_from_gdf_quadrature,
                     planar_transmittance, projected_area, projected_area_dir, sample_gdf,
                     vndf_eval, vndf_sample)
from .gp import (FirstHit, GpRealization, GridSpec, default_grid, empirical_transmittance,
                 empirical_vndf, ensemble_radiance, first_hit, multiplicativity_probe,
                 realize_gp)
from .errors import (ConfigError, DegenerateVisibilityError, GrazingSingularityError,
                     InternalConsistencyError, IoError, MacrofacetError, NumericFailureError,
                     ParameterDomainError, UnsupportedGeometryError)
from .image import RadianceImage, read_pfm, write_image, write_pfm, write_ppm
from .medium import (MacrofacetMedium, extinction, phase_eval, phase_pdf, phase_sample,
                     query_batch, query_batch_host)
from .ndf import KernelParams, NdfKind, RoughnessTriple, roughness_from_kernel
from .render import PathKeys, render, render_device, render_sharded, trace_path, trace_paths
from .rng import BatchRng, RandomStream, derive_bases, stream_base
from .scene import (Camera, DirectionalLight, Environment, PointLight, ShellPrimitive,
                    ShellScene, shell_intersect)
from .sdf import Box, Plane, Sphere
from .transport import EventKind, MediumEvent, sample_collision, transmittance_estimate, walk

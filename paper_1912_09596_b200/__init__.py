"""paper_1912_09596_b200 -- B200-native (sm_100a) empty-space-skipping build + render.

Drop-in for the reference package ``voxelskip`` (/root/reference/pkg/src/voxelskip/__init__.py):
the same public names, argument meanings, array layouts and exceptions, backed by
hand-written CUDA kernels in libvsb200.so (include/vsb200.h).  There is no CPU fallback.
"""

from .bench import (CSV_HEADER, INDEX_KINDS, BenchConfig, BenchRecord, build_index, index_kind,
                    load_dataset, load_tf, report_stats, run_benchmark, to_csv)
from .hybrid import HybridGrid, build_hybrid
from .kdtree import (BuildParams, CellBoxList, KdTree, SplitPlane, binned_best_plane, build_kdtree,
                     empty_kdtree, precompute_cell_boxes, sweep_best_plane)
from .lbvh import (BrickSet, Lbvh, MortonRangeError, build_lbvh, empty_lbvh, flag_bricks,
                   leaf_boxes, morton_decode, morton_encode)
from .render import (DEFAULT_DT, Camera, Frame, Ray, RaySegmentList, SpatialIndex, integrate,
                     render_float, render_frame, sample_count_of, traverse_grid, traverse_hybrid,
                     traverse_kd, traverse_lbvh, traverse_naive)
from .service import Reply, Session, handle_message
from .svt import (MacroGrid, SvtGrid, box_count, build_svt_grid, derive_macro_grid,
                  shrink_to_occupied)
from .volume import (Aabb, BinaryVolume, TransferFunction, UnsupportedFormatError, Volume,
                     VolumeFormatError, classify, gen_blobs, gen_menger, gen_shell, load_raw,
                     occupancy, quantize_scalar, save_raw)

__version__ = "0.1.0"

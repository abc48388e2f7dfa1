"""Generate golden vectors by running the UNMODIFIED reference (voxelskip) in the build container.

Usage (build container only; /root/reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference is imported from a scratch copy of /root/reference/pkg/src with NUMBA_CACHE_DIR
pointing at scratch, so numba's cache never writes into the read-only reference tree
(SURVEY.md §8c recipe).  Every fixture stores its inputs (u8 volumes / flag volumes, LUTs,
cameras) next to the reference outputs, so tests never need the generator or numba.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src/voxelskip")
REF_TESTS = Path("/root/reference/pkg/tests")


def _import_reference():
    scratch = Path(tempfile.gettempdir()) / "vsb200_ref_copy"
    if scratch.exists():
        shutil.rmtree(scratch)
    scratch.mkdir(parents=True)
    shutil.copytree(REF_SRC, scratch / "voxelskip")
    shutil.copy(REF_TESTS / "reference.py", scratch / "vs_reference_oracles.py")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(Path(tempfile.gettempdir()) / "vsb200_numba"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(scratch))
    import voxelskip  # noqa: F401
    import vs_reference_oracles  # noqa: F401

    return voxelskip, vs_reference_oracles


def u8_of(vs, v):
    """save_raw's quantiser (volume.py:275) -> u8, and the Volume load_raw would return."""
    q = np.rint(v.data.astype(np.float64) * 255.0).astype(np.uint8)
    return q, vs.Volume((q.astype(np.float64) / 255.0).astype(np.float32))


def band_tf(vs, lo, hi, a=0.5):
    lut = np.zeros((256, 4), np.float32)
    lut[:, 0] = np.linspace(0, 1, 256)
    lut[:, 1] = 0.5
    lut[:, 2] = np.linspace(1, 0, 256)
    lut[lo : hi + 1, 3] = a
    return vs.TransferFunction(lut)


def render_float(vs, v, tf, index, cam, dt=0.5, nearest=False):
    """Float RGBA oracle: _Traverser.run + _k_integrate."""
    from voxelskip.render import _CHUNK, _Traverser, _k_integrate

    field = np.ascontiguousarray(v.data, np.float32)
    lut = np.ascontiguousarray(tf.lut, np.float32)
    direction = np.asarray(cam.direction, np.float64)
    origins = cam.ray_origins()
    n = len(origins)
    trav = _Traverser(index, v.dims)
    rgba = np.zeros((n, 4))
    samples = np.zeros(n, np.int64)
    for s in range(0, n, _CHUNK):
        e = min(s + _CHUNK, n)
        segs, counts = trav.run(origins[s:e], direction)
        _k_integrate(origins[s:e], direction, segs, counts, field, lut, float(dt), nearest,
                     *v.dims, rgba[s:e], samples[s:e])
    return rgba.reshape(cam.height, cam.width, 4), samples.reshape(cam.height, cam.width)


def tree_dict(prefix, t, out):
    for f in ("lo", "hi", "left", "right"):
        out[f"{prefix}_{f}"] = np.asarray(getattr(t, f))
    if hasattr(t, "axis"):
        out[f"{prefix}_axis"] = np.asarray(t.axis)
        out[f"{prefix}_plane"] = np.asarray(t.plane)
    else:
        out[f"{prefix}_leaf_brick"] = np.asarray(t.leaf_brick)
        out[f"{prefix}_brick_coords"] = np.asarray(t.brick_coords)
    out[f"{prefix}_root"] = np.int64(t.root)
    out[f"{prefix}_height"] = np.int64(t.height())


KD_PARAMS = {
    "kd-shallow": dict(mode="shallow"),
    "kd-deep": dict(mode="deep"),
    "kd-deep-mls8": dict(mode="deep", max_leaf_size=8),
    "kd-deep-mls32": dict(mode="deep", max_leaf_size=32),
    "kd-deep-mls128": dict(mode="deep", max_leaf_size=128),
    "kd-binned-mls32": dict(mode="deep", max_leaf_size=32, builder="binned"),
    "kd-binned": dict(mode="deep", builder="binned"),
    "kd-binned-mls8": dict(mode="deep", max_leaf_size=8, builder="binned"),
}


def structures(vs, bits, out, prefix="", kd_kinds=tuple(KD_PARAMS), svt_bs=(32,)):
    b = vs.BinaryVolume(bits)
    out[prefix + "bits"] = np.packbits(bits.reshape(-1))
    out[prefix + "dims"] = np.asarray(bits.shape, np.int64)
    bs = vs.flag_bricks(b)
    out[prefix + "brick_coords_scan"] = bs.coords
    out[prefix + "brick_codes_scan"] = bs.codes
    tree_dict(prefix + "lbvh", vs.build_lbvh(bs), out)
    out[prefix + "grid16"] = vs.derive_macro_grid(b, 16).occupied
    for sbs in svt_bs:
        g = vs.build_svt_grid(b, sbs)
        out[prefix + f"svt{sbs}"] = g.tables
    cells = vs.precompute_cell_boxes(b, 8)
    for f in ("codes", "coords", "lo", "hi", "occupied"):
        out[prefix + f"cells8_{f}"] = getattr(cells, f)
    g = vs.build_svt_grid(b)
    for name in kd_kinds:
        tree_dict(prefix + name, vs.build_kdtree(g, vs.BuildParams(**KD_PARAMS[name])), out)
    return g


def main():
    vs, refo = _import_reference()
    import numba

    meta = dict(numpy=np.__version__, numba=numba.__version__, python=sys.version.split()[0])
    rng = np.random.default_rng(20240517)

    # ---- 1. blobs64: config-1 volume, five TFs, all structures, all renders ----
    v0 = vs.gen_blobs((64, 64, 64), 16, seed=7, sigma=3.0)
    u8, v = u8_of(vs, v0)
    tfs = {
        "ramp03": vs.TransferFunction.ramp(threshold=0.3),
        "ramp06": vs.TransferFunction.ramp(threshold=0.6),
        "ramp00": vs.TransferFunction.ramp(threshold=0.0),
        "opaque": vs.TransferFunction.opaque(),
        "band": band_tf(vs, 100, 140),
    }
    out = {"u8": u8, **{f"meta_{k}": np.asarray(x) for k, x in meta.items()}}
    for tname, tf in tfs.items():
        out[f"{tname}_lut"] = tf.lut
        plain = vs.classify(v, tf, dilate=False)
        out[f"{tname}_plain_bits"] = np.packbits(plain.bits.reshape(-1))
        out[f"{tname}_plain_count"] = np.int64(np.count_nonzero(plain.bits))
        out[f"{tname}_occupancy"] = np.float64(vs.occupancy(plain))
        dil = vs.classify(v, tf, dilate=True)
        kinds = tuple(KD_PARAMS) if tname == "ramp03" else ("kd-shallow", "kd-deep-mls32", "kd-binned-mls32")
        g = structures(vs, dil.bits, out, prefix=f"{tname}_", kd_kinds=kinds,
                       svt_bs=(32, 8) if tname == "ramp03" else (32,))
        if tname in ("ramp03", "band"):
            cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=96, height=64)
            out["cam_eye"] = np.asarray(cam.eye); out["cam_dir"] = np.asarray(cam.direction)
            out["cam_up"] = np.asarray(cam.up); out["cam_extent"] = np.float64(cam.extent)
            out["cam_origins"] = cam.ray_origins()
            idx = {
                "naive": None,
                "grid": vs.derive_macro_grid(dil, 16),
                "lbvh": vs.build_lbvh(vs.flag_bricks(dil)),
                "kd-shallow": vs.build_kdtree(g, vs.BuildParams(mode="shallow")),
                "kd-deep-mls32": vs.build_kdtree(g, vs.BuildParams(mode="deep", max_leaf_size=32)),
                "kd-binned-mls32": vs.build_kdtree(g, vs.BuildParams(mode="deep", max_leaf_size=32, builder="binned")),
                "hybrid": vs.build_hybrid(g, dil),
            }
            for kname, index in idx.items():
                rgba, samples = render_float(vs, v, tf, index, cam)
                fr = vs.render_frame(v, tf, index, cam)
                assert np.array_equal(fr.pixels, np.clip(np.floor(rgba * 255 + 0.5), 0, 255).astype(np.uint8))
                assert fr.sample_count == int(samples.sum())
                out[f"{tname}_render_{kname}_rgba"] = rgba
                out[f"{tname}_render_{kname}_samples"] = samples
                out[f"{tname}_render_{kname}_pixels"] = fr.pixels
            if tname == "ramp03":
                # single-ray traversal vectors (render.py:928-961)
                c = np.asarray(v.dims) / 2.0
                radius = float(np.linalg.norm(v.dims))
                rays_o, rays_d = [], []
                for _ in range(40):
                    u = rng.normal(size=3); u /= np.linalg.norm(u)
                    o = c + radius * u
                    d = rng.uniform(0.2, 0.8, size=3) * np.asarray(v.dims) - o
                    d /= np.linalg.norm(d)
                    rays_o.append(o); rays_d.append(d)
                # axis-aligned rays exercise the zero-direction branches
                for ax in range(3):
                    d = np.zeros(3); d[ax] = 1.0 if ax != 1 else -1.0
                    o = np.array([20.3, 31.7, 40.1]); o[ax] = -5.0 if d[ax] > 0 else 70.0
                    rays_o.append(o); rays_d.append(d)
                out["rays_o"] = np.asarray(rays_o); out["rays_d"] = np.asarray(rays_d)
                trav = {"naive": lambda r: vs.traverse_naive(r, v.dims),
                        "grid": lambda r: vs.traverse_grid(r, idx["grid"]),
                        "lbvh": lambda r: vs.traverse_lbvh(r, idx["lbvh"]),
                        "kd": lambda r: vs.traverse_kd(r, idx["kd-deep-mls32"]),
                        "hybrid": lambda r: vs.traverse_hybrid(r, idx["hybrid"])}
                for kname, fn in trav.items():
                    segs, counts = [], []
                    for o, d in zip(rays_o, rays_d):
                        s = fn(vs.Ray(origin=tuple(o), direction=tuple(d))).t
                        segs.append(s); counts.append(len(s))
                    out[f"trav_{kname}_counts"] = np.asarray(counts, np.int64)
                    out[f"trav_{kname}_segs"] = np.concatenate(segs).reshape(-1, 2) if segs else np.zeros((0, 2))
                # single-ray integrate
                ig_rgba, ig_samples = [], []
                for o, d in zip(rays_o, rays_d):
                    ray = vs.Ray(origin=tuple(o), direction=tuple(d))
                    segs = vs.traverse_naive(ray, v.dims)
                    ig_rgba.append(vs.integrate(ray, segs, v, tf))
                    ig_samples.append(vs.sample_count_of(ray, segs, v.dims))
                out["integrate_rgba"] = np.asarray(ig_rgba)
                out["integrate_samples"] = np.asarray(ig_samples, np.int64)
    np.savez_compressed(OUT / "blobs64.npz", **out)
    print("blobs64.npz", (OUT / "blobs64.npz").stat().st_size)

    # ---- 2. shell32 / menger2: the reference's own frame-equality scenes ----
    out = {}
    for scene, vol, w in (("shell", vs.gen_shell((32, 32, 32), radius=12.0, thickness=2.0), 64),
                          ("menger", vs.gen_menger(2), 64)):
        u8s, vv = u8_of(vs, vol)
        assert np.array_equal(vv.data, vol.data)
        out[f"{scene}_u8"] = u8s
        for tname, tf in (("opaque", vs.TransferFunction.opaque()), ("ramp", vs.TransferFunction.ramp())):
            out[f"{scene}_{tname}_lut"] = tf.lut
            dil = vs.classify(vv, tf, dilate=True)
            g = structures(vs, dil.bits, out, prefix=f"{scene}_{tname}_",
                           kd_kinds=("kd-shallow", "kd-deep", "kd-deep-mls32", "kd-binned-mls32"))
            cam = vs.Camera.orbit(vv.dims, 25.0, 20.0, width=w)
            idx = {"naive": None, "grid": vs.derive_macro_grid(dil, 16),
                   "lbvh": vs.build_lbvh(vs.flag_bricks(dil)),
                   "kd-deep-mls32": vs.build_kdtree(g, vs.BuildParams(mode="deep", max_leaf_size=32)),
                   "hybrid": vs.build_hybrid(g, dil)}
            for kname, index in idx.items():
                fr = vs.render_frame(vv, tf, index, cam)
                out[f"{scene}_{tname}_render_{kname}_pixels"] = fr.pixels
                out[f"{scene}_{tname}_render_{kname}_samples"] = np.int64(fr.sample_count)
            if tname == "ramp":
                fr = vs.render_frame(vv, tf, None, cam, interp="nearest")
                out[f"{scene}_{tname}_render_nearest_pixels"] = fr.pixels
                out[f"{scene}_{tname}_render_nearest_samples"] = np.int64(fr.sample_count)
    np.savez_compressed(OUT / "scenes.npz", **out)
    print("scenes.npz", (OUT / "scenes.npz").stat().st_size)

    # ---- 3. flag volumes straight from the reference test oracles (random / blocky / odd) ----
    out = {}
    cases = {
        "rand_64x48x40": refo.random_bits(rng, (64, 48, 40), density=0.02),
        "rand_20x17x9": refo.random_bits(rng, (20, 17, 9), density=0.1),
        "blocky48": refo.random_blocky_bits(rng, (48, 48, 48), block=8, density=0.15),
        "blocky_37x45x50": refo.random_blocky_bits(rng, (37, 45, 50), block=4, density=0.2),
        "sparse64": refo.random_bits(rng, (64, 64, 64), density=0.002),
    }
    for name, bits in cases.items():
        structures(vs, bits, out, prefix=f"{name}_", svt_bs=(32, 8, 4))
    np.savez_compressed(OUT / "bits.npz", **out)
    print("bits.npz", (OUT / "bits.npz").stat().st_size)

    # ---- 4. float volume (non-u8 field), ramp(0.2), naive + lbvh + kd render ----
    out = {}
    data = rng.random((16, 16, 16), dtype=np.float32)
    v = vs.Volume(data)
    tf = vs.TransferFunction.ramp(threshold=0.2)
    cam = vs.Camera.orbit(v.dims, 40.0, -20.0, width=32, height=24)
    dil = vs.classify(v, tf, dilate=True)
    out["f32_data"] = data
    out["f32_lut"] = tf.lut
    out["f32_dil_bits"] = np.packbits(dil.bits.reshape(-1))
    out["f32_plain_count"] = np.int64(np.count_nonzero(vs.classify(v, tf).bits))
    g = vs.build_svt_grid(dil)
    for kname, index in (("naive", None), ("lbvh", vs.build_lbvh(vs.flag_bricks(dil))),
                         ("kd", vs.build_kdtree(g, vs.BuildParams(mode="deep")))):
        rgba, samples = render_float(vs, v, tf, index, cam)
        out[f"f32_render_{kname}_rgba"] = rgba
        out[f"f32_render_{kname}_samples"] = samples
    # known answers from the reference tests
    snaps = []
    for lo, hi, bins, cs in ((8, 48, 4, 8), (0, 8, 4, 8), (0, 64, 2, 8), (3, 61, 4, 8), (5, 100, 7, 8),
                             (0, 1000, 4, 8), (17, 29, 4, 8), (1, 250, 5, 16)):
        p = vs.kdtree._snapped_positions(lo, hi, bins, cs)
        snaps.append([lo, hi, bins, cs, len(p)] + p + [0] * (8 - len(p)))
    out["snapped"] = np.asarray(snaps, np.int64)
    pow_tab = np.array([1.0 - (1.0 - float(a)) ** 0.5 for a in tfs["ramp03"].lut[:, 3]])
    out["corr_ramp03_dt05"] = pow_tab
    np.savez_compressed(OUT / "misc.npz", **out)
    print("misc.npz", (OUT / "misc.npz").stat().st_size)


EQUIV_KINDS = ("grid", "lbvh", "kd-shallow", "kd-deep-mls32", "kd-deep-mls128",
               "kd-binned-mls32", "hybrid")


def acceptance():
    """The reference's own acceptance datasets (pkg/tests/test_acceptance.py:206-234, criterion
    6; criterion 7's thin shell :237-259): 3 volumes x 2 TFs, every index kind's arrays and
    256x256 frames (pixels + sample counts) from the unmodified reference."""
    vs, _ = _import_reference()
    out = {}
    datasets = {
        "menger3": vs.gen_menger(3),
        "shell128": vs.gen_shell((128, 128, 128), radius=48.0, thickness=2.0),
        "blobs128": vs.gen_blobs((128, 128, 128), n=100, seed=7),
        "thinshell128": vs.gen_shell((128, 128, 128), radius=48.0, thickness=1.0),
    }
    tfs = {"opaque": vs.TransferFunction.opaque(), "ramp": vs.TransferFunction.ramp()}
    for dname, v in datasets.items():
        q = np.rint(v.data.astype(np.float64) * 255.0)
        if np.array_equal((q / 255.0).astype(np.float32), v.data):
            out[f"{dname}_u8"] = q.astype(np.uint8)   # u8-exact field: store the bins
        else:
            out[f"{dname}_f32"] = v.data                # float field (blobs): store it as is
        cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=256)
        for tname, tf in tfs.items():
            if dname == "thinshell128" and tname != "opaque":
                continue
            key = f"{dname}_{tname}"
            out[f"{tname}_lut"] = tf.lut
            out[f"{key}_plain_count"] = np.int64(np.count_nonzero(vs.classify(v, tf).bits))
            bits = vs.classify(v, tf, dilate=True)
            out[f"{key}_bits"] = np.packbits(bits.bits.reshape(-1))
            naive = vs.render_frame(v, tf, None, cam)
            out[f"{key}_naive_pixels"] = naive.pixels
            out[f"{key}_naive_samples"] = np.int64(naive.sample_count)
            kinds = ("kd-deep-mls32",) if dname == "thinshell128" else EQUIV_KINDS
            for kind in kinds:
                idx = vs.build_index(kind, bits)
                k = f"{key}_{kind}"
                if kind == "grid":
                    out[f"{k}_occupied"] = idx.occupied
                elif kind == "hybrid":
                    tree_dict(k, idx.tree, out)
                    out[f"{k}_occupied"] = idx.grid.occupied
                else:
                    tree_dict(k, idx, out)
                fr = vs.render_frame(v, tf, idx, cam)
                out[f"{k}_pixels"] = fr.pixels
                out[f"{k}_samples"] = np.int64(fr.sample_count)
            print(key, flush=True)
    np.savez_compressed(OUT / "acceptance.npz", **out)
    print("acceptance.npz", (OUT / "acceptance.npz").stat().st_size)


if __name__ == "__main__":
    if sys.argv[1:] == ["acceptance"]:
        acceptance()
    else:
        main()
        acceptance()

"""3DGS PLY loader (load_ply, scene_io.cpp:53-199) against the reference's own
loader, on files written by the reference's write_ply and by a header-flexible
writer here (extra properties, other elements first, lower SH degrees), plus
every error the reference raises. Host code only (no GPU)."""
import struct

import numpy as np
import pytest

from oracle.oracle import OracleError
from paper_2603_18707_b200 import abi, api


def _props(deg):
    n_rest = {0: 0, 1: 9, 2: 24, 3: 45}[deg]
    return (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"] +
            [f"f_rest_{i}" for i in range(n_rest)] + ["opacity", "scale_0", "scale_1", "scale_2",
                                                      "rot_0", "rot_1", "rot_2", "rot_3"])


def write_ply(path, rows, names, types=None, pre=b"", fmt="binary_little_endian 1.0", extra_header=""):
    """Minimal PLY writer: float32 vertex rows (n, len(names)) unless `types` says otherwise."""
    types = types or ["float"] * len(names)
    hdr = f"ply\nformat {fmt}\ncomment test\n{extra_header}element vertex {len(rows)}\n"
    hdr += "".join(f"property {t} {n}\n" for t, n in zip(types, names)) + "end_header\n"
    code = {"float": "f", "double": "d", "uchar": "B", "int": "i"}
    body = b"".join(struct.pack("<" + "".join(code[t] for t in types), *r) for r in rows)
    with open(path, "wb") as fh:
        fh.write(hdr.encode() + pre + body)


def _random_rows(n, deg, seed=0):
    rng = np.random.default_rng(seed)
    names = _props(deg)
    rows = rng.normal(0, 1, (n, len(names))).astype(np.float32)
    rows[:, names.index("opacity")] = rng.normal(0, 3, n)
    rows[:, names.index("scale_0"):names.index("scale_2") + 1] = rng.uniform(-6, -2, (n, 3))
    rows[0, names.index("rot_0"):names.index("rot_3") + 1] = 0.0   # degenerate quaternion -> identity
    return rows, names


def _same(a, b):
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.int64), b.view(np.int64))  # bitwise, incl. signed zeros


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_matches_reference_loader(reference, tmp_path, deg):
    rows, names = _random_rows(257, deg, seed=deg)
    p = tmp_path / "s.ply"
    write_ply(p, rows, names)
    ours, d1 = api.load_ply_splat3d(p)
    ref, d2 = reference.load_ply(p)
    assert d1 == d2 == deg
    _same(ours, ref)
    sc = api.load_ply(p)  # SoA view of the same decode
    assert sc.sh_degree == deg
    _same(sc.means, ref[:, 0:3])
    _same(sc.opacities, ref[:, 10])
    assert np.array_equal(sc.sh.reshape(-1, 48).astype(np.float64), ref[:, 11:59])


def test_round_trip_through_reference_writer(reference, tmp_path):
    splats, deg = api.synthetic_splat3d(1, 7)  # the reference's random scene
    p = tmp_path / "w.ply"
    reference.write_ply(splats, deg, p)
    ours, d1 = api.load_ply_splat3d(p)
    ref, d2 = reference.load_ply(p)
    assert d1 == d2 == 3
    _same(ours, ref)


def test_skips_other_elements_and_properties(reference, tmp_path):
    rows, names = _random_rows(33, 3, seed=5)
    # an extra uchar property in the middle, a double one at the end, and a
    # fixed-size element before the vertex element
    names2 = names[:4] + ["red"] + names[4:] + ["extra"]
    types = ["float"] * 4 + ["uchar"] + ["float"] * (len(names) - 4) + ["double"]
    rows2 = [tuple(r[:4]) + (7,) + tuple(r[4:]) + (1.5,) for r in rows.tolist()]
    p = tmp_path / "x.ply"
    hdr = "element camera 2\nproperty float a\nproperty int b\n"
    write_ply(p, rows2, names2, types, pre=struct.pack("<fifi", 1.0, 2, 3.0, 4), extra_header=hdr)
    ours, _ = api.load_ply_splat3d(p)
    ref, _ = reference.load_ply(p)
    _same(ours, ref)


def _status(fn):
    try:
        fn()
    except api.Error as e:
        return type(e).__name__
    except OracleError as e:
        return {abi.PS_IO_ERROR: "IoError", abi.PS_MALFORMED_HEADER: "MalformedHeader",
                abi.PS_UNSUPPORTED_FORMAT: "UnsupportedFormat", abi.PS_MISSING_PROPERTY: "MissingProperty",
                abi.PS_TRUNCATED_DATA: "TruncatedData"}.get(e.status, str(e.status))
    return "ok"


def _cases(tmp_path):
    rows, names = _random_rows(5, 3)
    out = {}

    def mk(name, **kw):
        p = tmp_path / f"{name}.ply"
        write_ply(p, kw.pop("rows", rows), kw.pop("names", names), **kw)
        return p
    out["missing_file"] = tmp_path / "nope.ply"
    out["ascii"] = mk("ascii", fmt="ascii 1.0")
    out["big_endian"] = mk("be", fmt="binary_big_endian 1.0")
    out["bad_version"] = mk("ver", fmt="binary_little_endian 2.0")
    no_op = [n for n in names if n != "opacity"]
    out["missing_opacity"] = mk("noop", rows=rows[:, [names.index(n) for n in no_op]], names=no_op)
    out["double_x"] = mk("dx", rows=[tuple(r) for r in rows.tolist()], names=names,
                         types=["double"] + ["float"] * (len(names) - 1))
    p = mk("trunc")
    data = p.read_bytes()
    p.write_bytes(data[:-10])
    out["truncated"] = p
    p = tmp_path / "nomagic.ply"
    p.write_bytes(b"plx\nformat binary_little_endian 1.0\nend_header\n")
    out["no_magic"] = p
    p = tmp_path / "noend.ply"
    p.write_bytes(b"ply\nformat binary_little_endian 1.0\n")
    out["no_end_header"] = p
    p = tmp_path / "token.ply"
    p.write_bytes(b"ply\nformat binary_little_endian 1.0\nbogus line\nend_header\n")
    out["bad_token"] = p
    p = tmp_path / "novert.ply"
    p.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement face 0\nend_header\n")
    out["no_vertex"] = p
    return out


def test_errors_match_reference(reference, tmp_path):
    for name, p in _cases(tmp_path).items():
        got = _status(lambda: api.load_ply_splat3d(p))
        want = _status(lambda: reference.load_ply(p))
        assert got == want and got != "ok", (name, got, want)


@pytest.mark.gpu
def test_checkpoint_renders_like_reference(gpu, reference, tmp_path):
    """A checkpoint straight into a device scene (ps_scene_load_ply) renders with
    the reference's counters and within 1e-5 of its image (C1-sized scene)."""
    from tests.helpers import camera, config
    splats, deg = api.synthetic_splat3d(3, 1, 10000)
    p = tmp_path / "c1.ply"
    reference.write_ply(splats, deg, p)
    ref_splats, _ = reference.load_ply(p)
    cam = camera(1, 256, 256, 0)
    cfg = config("poly1", api.CullingMode.OpacityAware, deg)
    ds = gpu.upload_ply(p)
    fb, ctr = gpu.render(ds, cam, cfg)
    rgb, tr, ctr_ref = reference.render(ref_splats, cam.to_struct(), cfg.to_struct())
    assert ctr.as_dict() == ctr_ref
    assert max(np.abs(fb.rgb - rgb).max(), np.abs(fb.transmittance - tr).max()) <= 1e-5
    ds.close()

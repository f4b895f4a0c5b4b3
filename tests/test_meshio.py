"""Mesh IO: the reference's text format
(mesh.py:280-371) through the native reader/writer, and the binary TALMESH1
format.  Goldens: files written by the reference's own save_mesh and the
error cases of its load_mesh (tests/golden/meshio/, oracle/gen_golden.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2403_08777_b200 as tb
from paper_2403_08777_b200.mesh import MeshFormatError, load_mesh, save_mesh, save_mesh_binary

G = Path(__file__).resolve().parent / "golden" / "meshio"


def test_save_is_byte_identical_to_reference_writer(tmp_path):
    """The reference's save_mesh output of two meshes, reproduced byte for byte."""
    gm = np.load(G / "meshes.npz")
    for name in ("box3x2x2", "odd"):
        m = tb.Mesh(coords=gm[f"{name}_coords"], connectivity=gm[f"{name}_conn"])
        out = tmp_path / f"{name}.txt"
        save_mesh(m, out)
        assert out.read_bytes() == (G / f"{name}.txt").read_bytes()


def test_load_reads_reference_files_exactly():
    gm = np.load(G / "meshes.npz")
    for name in ("box3x2x2", "odd"):
        m = load_mesh(G / f"{name}.txt")
        np.testing.assert_array_equal(m.coords, gm[f"{name}_coords"])
        np.testing.assert_array_equal(m.connectivity, gm[f"{name}_conn"])


def test_comments_blank_lines_and_reorientation():
    gm = np.load(G / "meshes.npz")
    with pytest.warns(UserWarning, match="re-oriented 2 inverted"):
        m = load_mesh(G / "commented_inverted.txt")
    np.testing.assert_array_equal(m.coords, gm["commented_inverted_coords"])
    np.testing.assert_array_equal(m.connectivity, gm["commented_inverted_conn"])


def test_format_errors_match_reference():
    """Each malformed file raises MeshFormatError with the reference's line
    number (the messages are the reference's up to quoting)."""
    cases = json.loads((G / "errors.json").read_text())
    for fname, want in cases.items():
        if want["type"] == "MeshFormatError":
            with pytest.raises(MeshFormatError) as ei:
                load_mesh(G / fname)
            assert ei.value.line == want["line"], (fname, str(ei.value), want)
            assert str(ei.value) == want["message"], (fname, str(ei.value), want)
        else:
            with pytest.raises(ValueError) as ei:
                load_mesh(G / fname)
            assert not isinstance(ei.value, MeshFormatError)


@pytest.mark.parametrize("fmt", ["text", "binary"])
def test_round_trip_exact(tmp_path, fmt):
    rng = np.random.default_rng(0)
    m = tb.generate_box_mesh(7, 5, 6)
    coords = m.coords + rng.uniform(-1e-3, 1e-3, m.coords.shape) * np.pi  # full-precision values
    m2 = tb.Mesh(coords=coords, connectivity=m.connectivity)
    p = tmp_path / f"m.{fmt}"
    (save_mesh if fmt == "text" else save_mesh_binary)(m2, p)
    r = load_mesh(p)
    np.testing.assert_array_equal(r.coords, m2.coords)
    np.testing.assert_array_equal(r.connectivity, m2.connectivity)


def test_binary_detects_corruption_and_truncation(tmp_path):
    m = tb.generate_box_mesh(3, 3, 3)
    p = tmp_path / "m.bin"
    save_mesh_binary(m, p)
    raw = bytearray(p.read_bytes())
    raw[100] ^= 0x10
    (tmp_path / "bad.bin").write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="hash"):
        load_mesh(tmp_path / "bad.bin")
    (tmp_path / "short.bin").write_bytes(p.read_bytes()[:-8])
    with pytest.raises(ValueError, match="complete"):
        load_mesh(tmp_path / "short.bin")
    with pytest.raises(OSError):
        load_mesh(tmp_path / "missing.txt")


def test_large_mesh_round_trip_binary_and_text(tmp_path):
    m = tb.generate_box_mesh(40, 40, 40)  # 384k tets
    for fn in (save_mesh, save_mesh_binary):
        p = tmp_path / fn.__name__
        fn(m, p)
        r = load_mesh(p)
        np.testing.assert_array_equal(r.coords, m.coords)
        np.testing.assert_array_equal(r.connectivity, m.connectivity)

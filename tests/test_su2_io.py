"""SU2 mesh I/O (mesh_io.cpp:127-309).

The native reader (im_su2_read) must return exactly what the reference's
read_su2 returns — nodes bit for bit, elements, markers with their node
lists — and fail on the same line with the same message; the writer must
produce the reference's bytes.  KATs restate tests/test_mesh_io.cpp."""
import os

import numpy as np
import pytest

import meshes as M
from paper_2107_13887_b200 import capi, workloads as W

UNIT_SQUARE = """NDIME= 2
NPOIN= 4
0.0 0.0
1.0 0.0
1.0 1.0
0.0 1.0
NELEM= 2
5 0 1 2
5 0 2 3
NMARK= 1
MARKER_TAG= wall
MARKER_ELEMS= 2
3 0 1
3 1 2
"""


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def same_mesh(a, b):
    assert a["dim"] == b["dim"]
    assert np.array_equal(a["nodes"].view(np.uint64), b["nodes"].view(np.uint64))
    for x, y in zip(a["elements"], b["elements"]):
        assert np.array_equal(np.asarray(x, np.int64), np.asarray(y, np.int64))
    assert [m["name"] for m in a["markers"]] == [m["name"] for m in b["markers"]]
    for ma, mb in zip(a["markers"], b["markers"]):
        assert np.array_equal(ma["nodes"], mb["nodes"])
        for x, y in zip(ma["elements"], mb["elements"]):
            assert np.array_equal(np.asarray(x, np.int64), np.asarray(y, np.int64))


def su2_text(dim, nodes, elements, markers, comments=False, crlf=False, order="std"):
    """An SU2 file in the reference layout, optionally with comments / blank
    lines / CRLF / reordered sections (all accepted by mesh_io.cpp)."""
    vtk = [3, 5, 9, 10, 12, 13, 14]
    k, o, c = elements
    sec = {}
    lines = [f"NELEM= {len(k)}"]
    for e in range(len(k)):
        lines.append(" ".join([str(vtk[k[e]])] + [str(int(v)) for v in c[o[e]:o[e + 1]]]))
        if comments and e % 7 == 3:
            lines.append("   % a comment line")
            lines.append("")
    sec["elem"] = lines
    lines = [f"NPOIN= {len(nodes)}"]
    for i, p in enumerate(nodes):
        lines.append(" ".join(repr(float(v)) for v in p[:dim]) + ("  % tail" if comments and i % 5 == 0 else ""))
    sec["poin"] = lines
    lines = [f"NMARK= {len(markers)}"]
    for name, (mk, mo, mc) in markers:
        lines += [f"MARKER_TAG= {name}", f"MARKER_ELEMS= {len(mk)}"]
        for e in range(len(mk)):
            lines.append(" ".join([str(vtk[mk[e]])] + [str(int(v)) for v in mc[mo[e]:mo[e + 1]]]))
    sec["mark"] = lines
    parts = ["% header comment", f"NDIME= {dim}"] if comments else [f"NDIME= {dim}"]
    for s in (["elem", "poin", "mark"] if order == "std" else ["mark", "poin", "elem"]):
        parts += sec[s]
    nl = "\r\n" if crlf else "\n"
    return nl.join(parts) + nl


def airfoil_case():
    w = W.cfg1(0.1)
    e = W.elements(w)
    ring = w.meta["ring"]
    # the innermost O-mesh ring as the wall marker (lines), the far ring as "far"
    nvol = w.meta["n_volume"]
    lines = [(M.LINE, [i, (i + 1) % ring]) for i in range(ring)]
    far0 = nvol - ring
    far = [(M.LINE, [far0 + i, far0 + (i + 1) % ring]) for i in range(ring)]
    nodes = w.nodes[:nvol]
    return nodes, e, [("wall", M.csr(lines)), ("far", M.csr(far))]


# ---- the reference's own KATs and error texts (CPU: reference only) -------------
def test_reference_kats(ref, tmp_path):
    m = ref.read_su2(write(tmp_path, "sq.su2", UNIT_SQUARE))
    assert m["dim"] == 2 and len(m["nodes"]) == 4 and list(m["markers"][0]["nodes"]) == [0, 1, 2]


# ---- product (needs the device for the coincident-node check) -------------------

@pytest.mark.gpu
def test_unit_square_and_marker_order(gpu, ref, tmp_path):  # test_mesh_io.cpp:35-55
    p = write(tmp_path, "sq.su2", UNIT_SQUARE)
    same_mesh(gpu.read_su2(p), ref.read_su2(p))
    text = UNIT_SQUARE.replace("3 0 1\n3 1 2\n", "3 2 1\n3 1 0\n")
    p = write(tmp_path, "order.su2", text)
    g = gpu.read_su2(p)
    assert list(g["markers"][0]["nodes"]) == [2, 1, 0]
    same_mesh(g, ref.read_su2(p))


BAD = {
    "ndime": "NDIME= x\n",
    "coord": "NDIME= 2\nNPOIN= 1\n0.0 zero\n",
    "few_coords": "NDIME= 2\nNPOIN= 1\n0.0\n",
    "kind": UNIT_SQUARE.replace("5 0 1 2", "7 0 1 2"),
    "not_allowed": UNIT_SQUARE.replace("5 0 1 2", "10 0 1 2 3"),
    "no_markers": "NDIME= 2\nNPOIN= 1\n0.0 0.0\nNELEM= 0\n",
    "range": UNIT_SQUARE.replace("5 0 2 3", "5 0 2 9"),
    "marker_range": UNIT_SQUARE.replace("3 1 2\n", "3 1 7\n"),
    "marker_kind": UNIT_SQUARE.replace("3 1 2\n", "5 1 2 0\n"),
    "needs": UNIT_SQUARE.replace("5 0 2 3", "5 0 2"),
    "bad_index": UNIT_SQUARE.replace("5 0 2 3", "5 0 x 3"),
    "type_id": UNIT_SQUARE.replace("5 0 2 3", "q 0 2 3"),
    "keyword": UNIT_SQUARE.replace("NELEM= 2", "NELEM 2"),
    "unknown": UNIT_SQUARE + "FOO= 1\n",
    "npoin_first": "NPOIN= 1\n0 0\n",
    "eof_points": "NDIME= 2\nNPOIN= 5\n0 0\n1 0\n",
    "eof_elems": UNIT_SQUARE.replace("NELEM= 2", "NELEM= 9"),
    "marker_tag": UNIT_SQUARE.replace("MARKER_TAG= wall", "MARKER= wall"),
    "marker_empty": UNIT_SQUARE.replace("MARKER_TAG= wall", "MARKER_TAG= "),
    "marker_elems": UNIT_SQUARE.replace("MARKER_ELEMS= 2", "MARKER_ELEMS= two"),
    "eof_marker": UNIT_SQUARE.replace("MARKER_ELEMS= 2", "MARKER_ELEMS= 3"),
    "duplicate": UNIT_SQUARE.replace("1.0 1.0", "1.0 0.0"),  # test_mesh_io.cpp:90-101
    "missing_elem": "NDIME= 2\nNPOIN= 1\n0.0 0.0\n",
    "two_errors": UNIT_SQUARE.replace("0.0 1.0", "0.0 bad").replace("5 0 1 2", "5 0 1 q"),
}


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(BAD))
def test_errors_match_reference(gpu, ref, tmp_path, case):
    p = write(tmp_path, "bad.su2", BAD[case])
    with pytest.raises(Exception) as r_exc:
        ref.read_su2(p)
    with pytest.raises(capi.ParseError) as g_exc:
        gpu.read_su2(p)
    assert str(g_exc.value) == str(r_exc.value)
    assert g_exc.value.line == r_exc.value.line
    if case == "duplicate":
        assert g_exc.value.line == 5 and "duplicate" in str(g_exc.value)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["plain", "comments", "crlf", "reordered"])
def test_airfoil_mesh_matches_reference(gpu, ref, tmp_path, variant):
    nodes, e, markers = airfoil_case()
    text = su2_text(2, nodes, e, markers, comments=variant == "comments", crlf=variant == "crlf",
                    order="reordered" if variant == "reordered" else "std")
    p = write(tmp_path, "af.su2", text)
    same_mesh(gpu.read_su2(p), ref.read_su2(p))


@pytest.mark.gpu
def test_3d_mesh_matches_reference(gpu, ref, tmp_path):
    rng = np.random.default_rng(3)
    bn, bel = M.box_grid(6, 5, 4)
    bn = bn + 0.01 * rng.standard_normal(bn.shape)
    quads = [(M.QUAD, [h[0], h[1], h[2], h[3]]) for _, h in bel[:30]]
    p = write(tmp_path, "box.su2", su2_text(3, bn, M.csr(bel), [("bottom", M.csr(quads))]))
    same_mesh(gpu.read_su2(p), ref.read_su2(p))


@pytest.mark.gpu
def test_writer_bytes_match_reference(gpu, ref, tmp_path):  # test_mesh_io.cpp:103-124
    nodes, e, markers = airfoil_case()
    src = write(tmp_path, "af.su2", su2_text(2, nodes, e, markers, comments=True))
    ours, theirs = str(tmp_path / "ours.su2"), str(tmp_path / "theirs.su2")
    m = gpu.read_su2(src)
    gpu.write_su2(ours, m["dim"], m["nodes"], m["elements"],
                  [(mk["name"], mk["elements"]) for mk in m["markers"]])
    ref.roundtrip_su2(src, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    same_mesh(gpu.read_su2(ours), m)  # round trip is exact


@pytest.mark.gpu
def test_python_mirror_su2(tmp_path):
    from paper_2107_13887_b200 import icemorph as im

    p = write(tmp_path, "sq.su2", UNIT_SQUARE)
    mesh = im.read_su2(p)
    assert mesh.num_nodes == 4 and mesh.num_elements == 2 and mesh.marker_nodes("wall") == [0, 1, 2]
    out = str(tmp_path / "back.su2")
    im.write_su2(mesh, out)
    text = open(out).read()
    assert text.startswith("NDIME= 2\nNELEM= 2\n5 0 1 2\n5 0 2 3\nNPOIN= 4\n0 0\n1 0\n")
    again = im.read_su2(out)
    assert again.nodes() == mesh.nodes() and again.marker_nodes("wall") == [0, 1, 2]

"""Graph files and build_csr against the reference itself.

load_graph (graph.cpp:68-161,180-184) is host parsing: its tests run without a GPU and
compare arrays, declared vertex counts, error kinds and messages with the reference
library (oracle/_ref). build_csr (graph.cpp:186-307) runs on the device: bit-exact CSR
arrays against the reference's build_csr on inputs with every merge rule exercised.
"""
import numpy as np
import pytest

import oracle as O
from paper_2411_11468_b200 import labelprop as lp

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref")

GOOD = {
    "mm_pattern_symmetric.mtx": (0, "%%MatrixMarket matrix coordinate pattern symmetric\n"
                                    "% a comment\n\n4 4 3\n2 1\n3 2\n4 4\n"),
    "mm_real_general.mtx": (0, "%%MatrixMarket Matrix Coordinate Real General\n5 3 4\n"
                               "1 2 0.5\n% mid comment\n2 1 1.25\n3 3 2\n5 1 3e-1\n"),
    "mm_integer.mtx": (0, "%%MatrixMarket matrix coordinate integer general\n3 3 2\n1 3 7\n3 1 7\n"),
    "el_plain.txt": (1, "# comment\n0 1\n1 2\n\n2 0 2.5\n% vertices 9\n3 3\n"),
    "el_declared_hash.txt": (1, "# vertices 6\n0 5 1\n5 0 1\n"),
    "el_empty.txt": (1, "# nothing here\n"),
}

BAD = {
    "mm_no_banner.mtx": (0, "1 1 1\n1 1\n"),
    "mm_array.mtx": (0, "%%MatrixMarket matrix array real general\n1 1\n1\n"),
    "mm_complex.mtx": (0, "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n"),
    "mm_hermitian.mtx": (0, "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n"),
    "mm_short_size.mtx": (0, "%%MatrixMarket matrix coordinate pattern general\n3 3\n"),
    "mm_zero_index.mtx": (0, "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n0 1\n"),
    "mm_outside.mtx": (0, "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n4 1\n"),
    "mm_truncated.mtx": (0, "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n"),
    "mm_bad_weight.mtx": (0, "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2 x\n"),
    "mm_neg_weight.mtx": (0, "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2 -1\n"),
    "mm_tokens.mtx": (0, "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2\n"),
    "mm_empty.mtx": (0, ""),
    "el_tokens.txt": (1, "0 1 2 3\n"),
    "el_bad_id.txt": (1, "0 a\n"),
    "el_big_id.txt": (1, "0 4294967295\n"),
    "el_zero_weight.txt": (1, "0 1 0\n"),
    "el_inf_weight.txt": (1, "0 1 inf\n"),
}


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


@needs_ref
@pytest.mark.parametrize("name", sorted(GOOD))
def test_load_graph_matches_reference(tmp_path, name):
    fmt, text = GOOD[name]
    p = _write(tmp_path, name, text)
    el = lp.load_graph(p, lp.FileFormat(fmt))
    u, v, w, nd = O.ref_load_graph(p, fmt)
    assert np.array_equal(el.u, u) and np.array_equal(el.v, v) and np.array_equal(el.w, w)
    assert (el.n_declared if el.n_declared is not None else -1) == nd


@needs_ref
@pytest.mark.parametrize("name", sorted(BAD))
def test_load_graph_errors_match_reference(tmp_path, name):
    fmt, text = BAD[name]
    p = _write(tmp_path, name, text)
    with pytest.raises(ValueError) as want:
        O.ref_load_graph(p, fmt)
    kind, msg = str(want.value).split(":", 1)
    err = lp.FormatError if kind == "F" else lp.ValidationError
    with pytest.raises(err) as got:
        lp.load_graph(p, lp.FileFormat(fmt))
    assert type(got.value) is err
    assert str(got.value) == msg


def test_load_graph_missing_file(tmp_path):
    with pytest.raises(lp.ValidationError, match="cannot open input file"):
        lp.load_graph(tmp_path / "nope.txt", lp.FileFormat.EdgeListText)


def _random_edges(rng, n, ne, loops=0.05, weighted=True):
    u = rng.integers(0, n, ne).astype(np.uint32)
    v = rng.integers(0, n, ne).astype(np.uint32)
    # repeat some listings in both directions and the same direction
    k = ne // 4
    u = np.concatenate([u, v[:k], u[k:2 * k]])
    v = np.concatenate([v, u[:k], v[k:2 * k]])
    sl = rng.random(u.size) < loops
    v[sl] = u[sl]
    w = (rng.random(u.size) * 3 + 0.1) if weighted else np.ones(u.size)
    return u.astype(np.uint32), v.astype(np.uint32), w


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("weighted", [True, False])
def test_build_csr_bit_exact(seed, weighted):
    rng = np.random.default_rng(seed)
    n = [20, 300, 5000, 70000][seed]
    u, v, w = _random_edges(rng, n, 8 * n, weighted=weighted)
    for nd in (None, n + 7):
        el = lp.EdgeList(u, v, w, nd)
        got = lp.build_csr(el, True)
        ref = O.RefGraph.from_edges(u, v, w, -1 if nd is None else nd, True)
        ro, rt, rw = ref.arrays()
        assert np.array_equal(got.offsets, ro) and np.array_equal(got.targets, rt)
        assert np.array_equal(got.weights.view(np.uint32), rw.view(np.uint32))


@needs_ref
@pytest.mark.gpu
def test_build_csr_directed_rules():
    # symmetric directed input (both directions, equal merged weights) builds; an
    # asymmetric one fails like the reference (the smallest offending edge is named).
    u = np.array([0, 1, 1, 2, 0, 1, 3], np.uint32)
    v = np.array([1, 0, 2, 1, 1, 0, 3], np.uint32)
    w = np.array([1.0, 1.5, 0.5, 0.5, 1.0, 0.5, 4.0])  # merged (0,1) = 2.0 = (1,0)
    el = lp.EdgeList(u, v, w, None)
    got = lp.build_csr(el, False)
    ro, rt, rw = O.RefGraph.from_edges(u, v, w, -1, False).arrays()
    assert np.array_equal(got.offsets, ro) and np.array_equal(got.targets, rt)
    assert np.array_equal(got.weights, rw)
    bad = lp.EdgeList(np.array([0, 1, 2], np.uint32), np.array([1, 0, 0], np.uint32),
                      np.ones(3), None)
    with pytest.raises(lp.ValidationError, match=r"not symmetric at edge \(2,0\)"):
        lp.build_csr(bad, False)
    with pytest.raises(lp.ValidationError, match="out of range for declared n=2"):
        lp.build_csr(lp.EdgeList(np.array([0], np.uint32), np.array([5], np.uint32),
                                 np.ones(1), 2), True)


@needs_ref
@pytest.mark.gpu
def test_load_graph_file_end_to_end(tmp_path):
    rng = np.random.default_rng(9)
    lines = ["%%MatrixMarket matrix coordinate real symmetric", "400 400 1500"]
    for _ in range(1500):
        a, b = rng.integers(1, 401, 2)
        lines.append(f"{max(a, b)} {min(a, b)} {rng.integers(1, 5) * 0.25}")
    p = _write(tmp_path, "g.mtx", "\n".join(lines) + "\n")
    dg = lp.DeviceGraph.load(p, lp.FileFormat.MatrixMarket)
    g = dg.download()
    u, v, w, nd = O.ref_load_graph(p, 0)
    ro, rt, rw = O.RefGraph.from_edges(u, v, w, nd, True).arrays()
    assert np.array_equal(g.offsets, ro) and np.array_equal(g.targets, rt)
    assert np.array_equal(g.weights, rw)
    r = dg.lpa(lp.LpaConfig(exec=lp.ExecMode.Synchronous))
    want, _ = O.port_lpa(O.PortGraph(ro, rt, rw), exec_mode=2)
    assert np.array_equal(r.labels, want)


# ---- chunk-parallel parsing: fuzzed files, many chunks, against the reference --------

def _fuzz_lines(rng, kind, n_lines):
    """Mostly valid lines of `kind` ('el', 'mm' or 'mem'), with comments, blanks, CRs and
    (sometimes) one bad line somewhere."""
    lines = []
    for i in range(n_lines):
        r = rng.random()
        if r < 0.03:
            lines.append("% a comment" if kind != "el" or rng.random() < 0.5 else "# c")
        elif r < 0.05:
            lines.append("   " if rng.random() < 0.5 else "")
        elif kind == "el":
            a, b = rng.integers(0, 500, 2)
            lines.append(f"{a} {b}" + (f" {rng.integers(1, 9) * 0.25}" if rng.random() < 0.5 else "")
                         + ("\r" if rng.random() < 0.05 else ""))
        elif kind == "mm":
            a, b = rng.integers(1, 301, 2)
            lines.append(f"{a}\t{b} {rng.integers(1, 9) * 0.5}")
        else:
            lines.append(f"{i}\t{rng.integers(0, n_lines)}")
    bad = {"el": ["0 x", "1 2 3 4", "7 4294967295", "3 4 -1", "% vertices 99999999999", "5"],
           "mm": ["1 2", "0 3 1", "400 1 1", "1 2 abc", "1 2 0"],
           "mem": ["x 1", "1 2 3", "1 2x", "99999999 1", "1 99999999"]}[kind]
    if rng.random() < 0.7:
        at = int(rng.integers(0, len(lines)))
        lines[at] = bad[int(rng.integers(0, len(bad)))]
    return lines


def _ours_or_error(fn):
    try:
        return "ok", fn()
    except (lp.FormatError, lp.ValidationError) as e:
        return ("F:" if type(e) is lp.FormatError else "V:") + str(e), None


def _refs_or_error(fn):
    try:
        return "ok", fn()
    except ValueError as e:
        return str(e), None


@needs_ref
@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("kind", ["el", "mm"])
def test_graph_file_chunks_match_reference(tmp_path, monkeypatch, seed, kind):
    monkeypatch.setenv("NULPA_TEXT_CHUNK_BYTES", str(64 + 97 * seed))  # many small chunks
    rng = np.random.default_rng(1000 * seed + len(kind))
    body = _fuzz_lines(rng, kind, 400)
    if kind == "mm":
        nnz = int(rng.integers(300, 420))  # sometimes short, sometimes trailing junk
        text = f"%%MatrixMarket matrix coordinate real general\n% c\n300 300 {nnz}\n"
    else:
        text = "% vertices 600\n" if seed % 2 else ""
    p = tmp_path / f"g.{kind}"
    p.write_text(text + "\n".join(body) + ("\n" if seed % 3 else ""))
    fmt = 0 if kind == "mm" else 1
    got, el = _ours_or_error(lambda: lp.load_graph(p, lp.FileFormat(fmt)))
    want, ref = _refs_or_error(lambda: O.ref_load_graph(p, fmt))
    assert got == want
    if el is not None:
        u, v, w, nd = ref
        assert np.array_equal(el.u, u) and np.array_equal(el.v, v) and np.array_equal(el.w, w)
        assert (el.n_declared if el.n_declared is not None else -1) == nd


@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_read_membership_chunks_match_reference(tmp_path, monkeypatch, seed):
    monkeypatch.setenv("NULPA_TEXT_CHUNK_BYTES", str(48 + 61 * seed))
    rng = np.random.default_rng(seed)
    n = 300
    lines = _fuzz_lines(rng, "mem", n)
    if seed % 4 == 1:  # a duplicate vertex
        lines.append(f"{int(rng.integers(0, n))}\t0")
    if seed % 4 == 2:  # a missing vertex
        lines = [ln for ln in lines if not ln.startswith(f"{n - 7}\t")]
    p = tmp_path / "m.tsv"
    p.write_text("\n".join(lines) + "\n")
    got, lab = _ours_or_error(lambda: lp.read_membership(p, n))
    want, ref = _refs_or_error(lambda: O.ref_read_membership(p, n))
    assert got == want
    if lab is not None:
        assert np.array_equal(lab, ref)


@needs_ref
@pytest.mark.parametrize("weighted", [False, True])
def test_write_edge_list_bytes_match_reference(tmp_path, monkeypatch, weighted):
    rng = np.random.default_rng(5)
    n = 3000
    u, v, w = _random_edges(rng, n, 6 * n, weighted=weighted)
    ref = O.RefGraph.from_edges(u, v, w, n + 5, True)
    ro, rt, rw = ref.arrays()
    O.ref_write_edge_list(ref, tmp_path / "ref.txt")
    g = lp.CsrGraph(ro, rt, rw)
    lp.write_edge_list(g, tmp_path / "ours.txt")
    assert (tmp_path / "ours.txt").read_bytes() == (tmp_path / "ref.txt").read_bytes()
    with pytest.raises(lp.ValidationError, match="cannot open output file"):
        lp.write_edge_list(g, tmp_path / "no" / "such" / "dir.txt")


@needs_ref
@pytest.mark.gpu
def test_write_membership_bytes_match_reference(tmp_path):
    rng = np.random.default_rng(2)
    for n in (0, 1, 10, 12345, 3 * (1 << 20) + 17):
        lab = rng.integers(0, max(n, 1), n).astype(np.uint32)
        if n > 5:
            lab[:3] = [0, n - 1, 9]
        lp.write_membership(tmp_path / "ours.tsv", lab)
        O.ref_write_membership(tmp_path / "ref.tsv", lab)
        assert (tmp_path / "ours.tsv").read_bytes() == (tmp_path / "ref.tsv").read_bytes()
        if n:
            assert np.array_equal(lp.read_membership(tmp_path / "ours.tsv", n), lab)

"""Host-side checks of the C-ABI library (no GPU needed): the shared library
builds, loads, and exports every function include/mgdtn.h declares; the
ctypes binding declares exactly those names; the product path never imports
the oracle and has no CPU fallback."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mgdtn.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(mg_[a-z_0-9]+)\s*\(", src))


@pytest.fixture(scope="module")
def lib():
    from paper_1811_09909_b200 import build
    build.build()
    from paper_1811_09909_b200.mgdtn import load_library
    return load_library()


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for n in ("mg_build_hierarchy", "mg_setup_dtn", "mg_apply", "mg_vcycle", "mg_pcg_solve"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_matches_header():
    from paper_1811_09909_b200.mgdtn import _SIGS
    assert set(_SIGS) == _declared()


def test_host_only_calls_without_gpu(lib):
    """mg_build_hierarchy / mg_workspace_bytes / mg_level_info are host-only."""
    import ctypes as C
    from paper_1811_09909_b200.mgdtn import mg_quad_mesh
    mesh = mg_quad_mesh(256, 256, 0.0, 0.0, 1.0 / 256)
    ctx = C.c_void_p()
    assert lib.mg_build_hierarchy(C.byref(mesh), 4, 0, None, None, C.byref(ctx)) == 0
    nl = C.c_int32()
    assert lib.mg_num_levels(ctx, C.byref(nl)) == 0
    assert nl.value == 9          # p-level + 256 -> 2 (9 levels)
    nb = C.c_size_t()
    assert lib.mg_workspace_bytes(ctx, C.byref(nb)) == 0
    # packed fine DtN: 65536 * 210 doubles = 110 MB, plus vectors / coarse levels
    assert 110e6 < nb.value < 1e9
    nx, ny, p, nd = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
    assert lib.mg_level_info(ctx, 9, C.byref(nx), C.byref(ny), C.byref(p), C.byref(nd)) == 0
    assert (nx.value, p.value, nd.value) == (256, 4, 657920)
    assert lib.mg_level_info(ctx, 1, C.byref(nx), C.byref(ny), C.byref(p), C.byref(nd)) == 0
    assert (nx.value, p.value) == (2, 1)
    # errors are statuses, never aborts
    assert lib.mg_level_info(ctx, 10, C.byref(nx), C.byref(ny), C.byref(p), C.byref(nd)) == -1
    assert lib.mg_setup_dtn(ctx, None, None, None, None) in (-1, -8)
    lib.mg_destroy(ctx)
    bad = mg_quad_mesh(7, 8, 0.0, 0.0, 0.1)
    assert lib.mg_build_hierarchy(C.byref(bad), 1, 0, None, None, C.byref(ctx)) == -2
    assert lib.mg_build_hierarchy(C.byref(mesh), 5, 0, None, None, C.byref(ctx)) == -1


def test_level_counts_match_survey(lib):
    import ctypes as C
    from paper_1811_09909_b200.mgdtn import mg_quad_mesh
    for n, p, want in ((8, 1, 3), (256, 4, 9), (1024, 2, 11), (512, 3, 10), (4096, 4, 13)):
        mesh = mg_quad_mesh(n, n, 0.0, 0.0, 1.0 / n)
        ctx = C.c_void_p()
        assert lib.mg_build_hierarchy(C.byref(mesh), p, 0, None, None, C.byref(ctx)) == 0
        nl = C.c_int32()
        lib.mg_num_levels(ctx, C.byref(nl))
        assert nl.value == want, (n, p, nl.value)
        lib.mg_destroy(ctx)


def test_nonsymmetric_build_host_only(lib):
    """MG_BUILD_NONSYMMETRIC (IIPG-H / NIPG-H, Eq. IPG_H): full element maps (m*m
    doubles, 400 at p=4 vs 210 packed), bad flags refused, no partition."""
    import ctypes as C
    from paper_1811_09909_b200.mgdtn import mg_partition, mg_quad_mesh
    mesh = mg_quad_mesh(256, 256, 0.0, 0.0, 1.0 / 256)
    sizes = []
    for flags in (0, 1):
        ctx = C.c_void_p()
        assert lib.mg_build_hierarchy_ex(C.byref(mesh), 4, 0, None, flags, None, C.byref(ctx)) == 0
        nb = C.c_size_t()
        assert lib.mg_workspace_bytes(ctx, C.byref(nb)) == 0
        sizes.append(nb.value)
        lib.mg_destroy(ctx)
    fine_packed, fine_full = 65536 * 210 * 8, 65536 * 400 * 8
    # the symmetric context also holds the orbit records of its two finest levels
    # (R9: 33 + 7 values per element, D_e^-1 orbits) instead of their packed D_e^-1
    orbit = 65536 * 8 * (33 + 7) + 2 * 131584 * 8 * (9 + 2)
    assert sizes[1] - sizes[0] >= fine_full - fine_packed - orbit
    ctx = C.c_void_p()
    assert lib.mg_build_hierarchy_ex(C.byref(mesh), 4, 0, None, 2, None, C.byref(ctx)) == -1
    part = mg_partition(0, 2, 2, 1, None, 0, None)
    assert lib.mg_build_hierarchy_ex(C.byref(mesh), 4, 0, C.byref(part), 1, None, C.byref(ctx)) == -9


def _imports(path):
    tree = ast.parse(open(path).read())
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            yield from (a.name for a in node.names)
        elif isinstance(node, ast.ImportFrom):
            yield node.module or ""


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1811_09909_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert not any(m.startswith("oracle") for m in _imports(os.path.join(pkg, fn))), fn
    # and neither the oracle nor the input generators import the product path
    for d in ("oracle", "workloads"):
        for fn in os.listdir(os.path.join(ROOT, d)):
            if fn.endswith(".py"):
                mods = list(_imports(os.path.join(ROOT, d, fn)))
                assert not any("paper_1811_09909_b200" in m for m in mods), fn
                if d == "workloads":
                    assert not any(m.startswith("oracle") for m in mods), fn


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1811_09909_b200 import MGError, MGSolver
    with pytest.raises(MGError):
        MGSolver(8, p=1)


def test_bench_flags_not_shadowed():
    """bench.py main(): the nonsymmetric-scheme flag `ns` is assigned once (a later
    reuse of the name once relabelled the default PCG line as GMRES)."""
    src = open(os.path.join(ROOT, "bench.py")).read()
    tree = ast.parse(src)
    main = next(n for n in tree.body if isinstance(n, ast.FunctionDef) and n.name == "main")
    targets = [t.id for node in ast.walk(main) if isinstance(node, ast.Assign)
               for t in node.targets if isinstance(t, ast.Name)]
    assert targets.count("ns") == 1, targets.count("ns")


def test_agglomerate_seeds_rejects_bad_arguments_on_the_host(lib):
    """mg_agglomerate_seeds validates sizes / pointers before touching the device."""
    import ctypes as C
    bad = C.c_int64(7)
    dummy = C.c_void_p(16)
    assert lib.mg_agglomerate_seeds(0, 4, dummy, dummy, dummy, 1, dummy, 3, dummy, dummy, None,
                                    None, None, C.byref(bad)) == -1
    assert bad.value == -1
    assert lib.mg_agglomerate_seeds(4, 4, dummy, dummy, dummy, 1, dummy, 1, dummy, dummy, None,
                                    None, None, None) == -1          # nlev < 2
    assert lib.mg_agglomerate_seeds(4, 4, None, dummy, dummy, 1, dummy, 3, dummy, dummy, None,
                                    None, None, None) == -1          # NULL edge_elem
    assert lib.mg_agglomerate_seeds(4, 4, dummy, dummy, dummy, 1, dummy, 3, dummy, dummy, dummy,
                                    None, None, None) == -1          # medge without nmedge
    assert lib.mg_agglomerate_seeds(4, 4, dummy, dummy, dummy, 1 << 20, dummy, 8, dummy, dummy,
                                    None, None, None, None) == -1    # ids beyond int32

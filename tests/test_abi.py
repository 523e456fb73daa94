"""CPU-side checks of the boundary: libdmoe.so loads and exports every symbol include/dmoe.h declares."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dmoe.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int32_t|size_t|dmoe_status|void)\s+(dmoe_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    for n in ["dmoe_gate_scores", "dmoe_beam_topk", "dmoe_dispatch", "dmoe_expert_ffn_fwd",
              "dmoe_expert_ffn_bwd", "dmoe_combine", "dmoe_combine_bwd", "dmoe_gate_bwd"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2002_04013_b200", "libdmoe.so"))
    for n in declared_symbols():
        assert hasattr(lib, n), n


def test_binding_exposes_same_names():
    import paper_2002_04013_b200 as P
    for n in declared_symbols():
        if n in ("dmoe_last_error",):
            continue
        assert hasattr(P, n), n


def test_validation_errors_without_gpu():
    """Argument validation is synchronous and needs no device (include/dmoe.h conventions)."""
    import paper_2002_04013_b200 as P
    from paper_2002_04013_b200 import _lib as L
    g = P.grid(2, 4, 4)
    assert L._L.dmoe_gate_scores(None, 1, 8, 64, None, None, L.grid(5, 4, 4), None, None, 0, None) == -2   # d > 4
    assert L._L.dmoe_gate_scores(None, 1, 8, 64, None, None, L.grid(2, 4, 17), None, None, 0, None) == -2  # k > 16
    assert L._L.dmoe_gate_scores(None, 1, 8, 60, None, None, g, None, None, 0, None) == -2                  # D % 8
    assert L._L.dmoe_gate_scores(None, 7, 8, 64, None, None, g, None, None, 0, None) == -1                  # dtype
    assert L._L.dmoe_gate_scores(None, 1, 8, 64, None, None, g, None, None, 0, None) == -1                  # null
    assert b"null pointer" in L._L.dmoe_last_error()
    assert P.dmoe_workspace_bytes(4096, 256, 1024, g, 16, 16384) > 16384 * 1024 * 2


def _prototypes():
    """name -> parameter count of every function prototype in include/dmoe.h."""
    src = open(os.path.join(ROOT, "include", "dmoe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"(?:const char\*|int32_t|size_t|dmoe_status|void)\s+(dmoe_\w+)\s*\(([^;{]*?)\)\s*;", src):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_binding_signatures_match_the_header():
    """The ctypes argtypes of every bound call have the header's parameter count (ABI drift check)."""
    from paper_2002_04013_b200 import _lib as L
    protos = _prototypes()
    assert "dmoe_expert_ffn_fwd" in protos and "dmoe_expert_ffn_bwd" in protos
    checked = 0
    for name, n in protos.items():
        f = getattr(L._L, name, None)
        if f is None or f.argtypes is None:
            continue
        assert len(f.argtypes) == n, (name, len(f.argtypes), n)
        checked += 1
    assert checked >= 10

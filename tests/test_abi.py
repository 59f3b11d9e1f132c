"""The C-ABI library builds, loads and exports every symbol include/roast.h declares (no GPU)."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "roast.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(roast_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for n in ["roast_create", "roast_register_linear", "roast_register_embedding", "roast_linear_fwd",
              "roast_linear_bwd", "roast_embedding_fwd", "roast_embedding_bwd", "roast_grad_allreduce"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2207_10702_b200 import build, roast
    lib = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib], text=True)
    exported = set(re.findall(r"\bT (roast_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    assert set(roast.EXPORTS) == set(declared_functions())


def test_library_has_sm100a_code_and_tensor_core_instructions():
    from paper_2207_10702_b200 import build
    lib = build.build()
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], text=True)
    assert "sm_100a" in subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib], text=True)
    assert "FFMA" in sass


def test_config_defaults_without_gpu():
    from paper_2207_10702_b200 import roast
    cfg = roast.roast_config_default()
    assert (cfg.C, cfg.align_elems, cfg.tile_layout, cfg.mapping, cfg.use_sign, cfg.deterministic) == \
        (1.0, 8, 0, 0, 1, 0)
    assert roast._lib.roast_status_str(4) == b"bounds error"

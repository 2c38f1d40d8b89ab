"""CPU-side checks of the C ABI boundary: the library builds for sm_100a, loads, and exports every
entry point include/osmpm.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "osmpm.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(osmpm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_09097_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("osmpm_subdomain_create", "osmpm_p2g", "osmpm_newton_hvp", "osmpm_g2p", "osmpm_transmit",
              "osmpm_schwarz_substep"):
        assert f in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert set(declared_functions()) <= exported


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string(libpath):
    lib = ctypes.CDLL(libpath)
    lib.osmpm_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.osmpm_version()


def test_library_is_built_from_the_current_sources(libpath):
    """build() embeds the sha256 of csrc/ + include/ + flags; the loaded library must carry the hash of
    the sources in the tree (no stale binary from another checkout)."""
    from paper_2605_09097_b200 import build
    lib = ctypes.CDLL(libpath)
    lib.osmpm_version.restype = ctypes.c_char_p
    assert lib.osmpm_version().decode().endswith("src " + build.source_hash())


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2605_09097_b200 import osmpm
    monkeypatch.setattr(osmpm, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(osmpm, "_lib", None)
    with pytest.raises(ImportError):
        osmpm.lib()

"""The C-ABI library loads on a CPU-only box and exports every symbol the header declares;
no compute calls are made here."""

import ctypes
import os
import re
import subprocess

from paper_2505_12658_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hydra_sm100.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hy_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_are_bound():
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(_lib.EXPORTED_SYMBOLS) == syms


def test_library_loads_and_exports():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.hy_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hy_[a-z0-9_]+)", out))
    assert set(header_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    # tcgen05 MMA + TMA loads + TMEM loads prove the Blackwell-native GEMM path
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_host_modules_do_not_map_the_library():
    """The reference arm of bench.py (epdsim + the CPU port) imports the package's host
    modules; the .so must only load on first device use (GpuCluster / InstanceRuntime /
    DeviceWeights), so that arm never maps it."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2505_12658_b200 as P\n"
            "from paper_2505_12658_b200 import _lib, inputs, shapes, planner, weights\n"
            "import oracle.cpu_executor, bench\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert _lib._lib is None and 'libhydra_sm100' not in maps\n"
            "print('ok')\n") % ROOT
    out = subprocess.run(["python", "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert out.stdout.strip() == "ok", out.stderr

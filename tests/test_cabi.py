"""The C-ABI libraries load and export every symbol their headers declare
(no compute calls: this runs on the CPU-only container too)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2504_08795_b200" / "lib"


def _declared(header: str) -> set[str]:
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(daris_[a-z0-9_]+)\s*\(", text))


@pytest.mark.parametrize("lib,headers", [("libdaris_core.so", ["daris.h"]),
                                          ("libdaris_gpu.so", ["daris_kernels.h", "daris_exec.h"])])
def test_library_exports_header_symbols(lib, headers):
    path = LIB / lib
    assert path.exists(), f"{path} not built"
    if lib == "libdaris_gpu.so":
        ctypes.CDLL(str(LIB / "libdaris_core.so"), mode=ctypes.RTLD_GLOBAL)
    so = ctypes.CDLL(str(path))
    declared = set().union(*(_declared(h) for h in headers))
    assert declared, "no declarations parsed"
    missing = [name for name in sorted(declared) if not hasattr(so, name)]
    assert not missing, f"{lib} lacks {missing}"


def test_python_binding_covers_core_abi():
    from paper_2504_08795_b200 import _core
    declared = _declared("daris.h")
    bound = set(_core.EXPORTED_SYMBOLS)
    # every bound name is declared, and the ABI subset the drop-in API uses is bound
    assert bound <= declared
    for name in ("daris_create", "daris_release", "daris_dispatch", "daris_complete", "daris_sim_run",
                 "daris_trace_run"):
        assert name in bound


def test_py_sum_matches_cpython_builtin():
    import random
    from paper_2504_08795_b200 import _core
    L = _core.lib()
    rng = random.Random(3)
    for _ in range(300):
        n = rng.randint(0, 12)
        vals, flags = [], []
        for _ in range(n):
            if rng.random() < 0.3:
                v = rng.randint(-50, 200)
                vals.append(v)
                flags.append(1)
            else:
                v = rng.choice([1e16, -1e16, 0.1, 1e-9, rng.uniform(-5, 5), rng.uniform(0, 1e-3)])
                vals.append(v)
                flags.append(0)
        arr = (ctypes.c_double * max(1, n))(*[float(v) for v in vals])
        fl = (ctypes.c_int32 * max(1, n))(*flags)
        assert L.daris_py_sum(arr, fl, n) == float(sum(vals)), vals


def test_conv_tile_width_rule():
    """daris_conv_plan (host-only): 64-wide tiles when the 128-wide grid leaves
    resident CTA slots (3 per planned SM) idle and the 64-wide grid fits in them;
    128-wide otherwise (large batches keep their plans)."""
    from paper_2504_08795_b200 import kernels as K

    def bn(shape, cout, k, budget):
        return K.conv_plan(K.conv_desc(shape, cout, k, k, 1, k // 2, sm_budget=budget)).block_n

    # 7 M tiles x 4 = 28 < 3*23 and 56 <= 69 -> 64 wide
    assert bn((1, 28, 28, 128), 512, 1, 23) == 64
    # 28 x 2 = 56 < 69 but the 64-wide grid (112) would overflow 69 slots -> 128
    assert bn((1, 56, 56, 64), 256, 1, 23) == 128
    # batch 64 on the whole GPU: 256 tiles of 128 -> stays 128
    assert bn((64, 14, 14, 256), 256, 3, 148) == 128


def test_conv_flat_m_tiles_for_1x1():
    """daris_conv_plan (host-only): 1x1 stride-1 convolutions tile M as a flat
    [pixels, channels] GEMM when that needs fewer 128-row tiles than whole image
    rows per tile; spatial kernels and batch-1 shapes that gain nothing keep
    their per-image plans."""
    from paper_2504_08795_b200 import kernels as K

    def plan(shape, cout, k, stride=1, budget=148):
        return K.conv_plan(K.conv_desc(shape, cout, k, k, stride, k // 2, sm_budget=budget))

    assert plan((64, 7, 7, 512), 2048, 1).tiles_m == 25        # 3136 px: 64 images -> 25 tiles
    assert plan((64, 14, 14, 256), 1024, 1).tiles_m == 98      # 12544 px = 98 x 128
    assert plan((64, 56, 56, 64), 256, 1).tiles_m == 1568      # 2 rows of 56 (112) -> 128 flat rows
    assert plan((64, 14, 14, 256), 256, 3).tiles_m == 128      # 3x3: per-image row tiles (9 + 5 rows)
    assert plan((1, 14, 14, 1024), 256, 1, budget=32).tiles_m == 2   # batch 1: no gain, unchanged
    assert plan((1, 7, 7, 512), 2048, 1, budget=32).tiles_m == 1
    assert plan((1, 56, 56, 256), 64, 1, budget=32).tiles_m == 28  # one wave of 87.5 %-full tiles: kept
    # the fused downsample (1x1 stride 2 over a 2x larger x2): images stack along H, rows stay 7 wide
    dual = K.conv_desc((64, 7, 7, 512), 2048, 1, 1, 1, 0, sm_budget=148, x2_shape=(64, 14, 14, 1024), stride2=2)
    assert K.conv_plan(dual).tiles_m == 25                      # 448 rows of 7 in boxes of 18 rows (was 64)
    # 3x3 on 7x7 maps: whole images per tile (2 x 49 rows), batch 1 unchanged
    assert plan((64, 7, 7, 512), 512, 3).tiles_m == 32
    assert plan((3, 7, 7, 512), 512, 3).tiles_m == 2
    assert plan((1, 7, 7, 512), 512, 3, budget=32).tiles_m == 1
    assert plan((8, 14, 14, 256), 256, 3).tiles_m == 16         # 196 px > 64: one image per tile, 2 tiles each


def test_gpu_library_is_tcgen05_tma_sm100a():
    """The built kernel library is sm_100a SASS that issues tcgen05 MMAs
    (UTCHMMA) and TMA loads/stores (UTMALDG/UTMASTG), and the conv kernels keep
    the 96-register cap that admits 3 resident CTAs per SM (cuobjdump, no GPU)."""
    import re
    import shutil
    import subprocess
    from pathlib import Path
    import pytest
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    lib = Path(__file__).resolve().parents[1] / "paper_2504_08795_b200" / "lib" / "libdaris_gpu.so"
    sass = subprocess.run([cuobjdump, "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in sass
    for mnemonic in ("UTCHMMA", "UTMALDG", "UTMASTG"):
        assert mnemonic in sass, mnemonic
    # the CTA-pair conv kernel: 2-SM MMAs, 2-SM TMA loads, multicast commits
    for mnemonic in ("UTCHMMA.2CTA", "UTMALDG.4D.2CTA", "UTCBAR.2CTA.MULTICAST"):
        assert mnemonic in sass, mnemonic
    # the classifier layers run on the tensor cores too: every linear_tc_kernel
    # instantiation issues tcgen05 MMAs
    funcs = re.split(r"\n\s*Function : ", sass)
    lin = [f for f in funcs if f.startswith("_ZN5daris16linear_tc_kernel")]
    assert len(lin) == 5 and all("UTCHMMA" in f for f in lin), len(lin)
    res = subprocess.run([cuobjdump, "-res-usage", str(lib)], capture_output=True, text=True, check=True).stdout
    regs = [int(r) for r in re.findall(r"conv_igemm_tc_kernel\S*:\s*\n\s*REG:(\d+)", res)]
    assert regs and max(regs) <= 96, regs


def test_partition_layout_covers_the_device_os_times():
    """daris_partition_layout (the executor's green-partition rule) over B200's
    units [28-SM remainder, 15 x 8-SM groups]: for every C4 cell (OS <= N_c) the
    partitions together cover the device about OS times, every unit is used,
    each partition is within the largest unit of ceil_even(OS * 148 / N_c), and OS = 1
    tiles the device exactly when the remainder fits one partition."""
    import math
    from paper_2504_08795_b200 import _core
    units = [28] + [8] * 15

    def ceil_even(x):
        c = math.ceil(x - 1e-9)
        return c + (c % 2)
    for os_ in (1.0, 1.5, 2.0, 3.0):
        for nc in (2, 4, 8):
            if os_ > nc:
                continue
            spc = min(148, ceil_even(os_ * 148 / nc))
            lay = _core.partition_layout(nc, spc, units)
            covered = [0] * len(units)
            for first, taken, sms in lay:
                assert sms == sum(units[(first + q) % len(units)] for q in range(taken))
                assert abs(sms - spc) <= max(units), (os_, nc, spc, lay)   # within the largest unit
                for q in range(taken):
                    covered[(first + q) % len(units)] += 1
            assert min(covered) >= 1, (os_, nc, covered)          # every SM is in some partition
            total = sum(s for _, _, s in lay)
            assert abs(total - os_ * 148) <= 0.12 * os_ * 148, (os_, nc, total)
            if os_ == 1.0 and nc <= 4:
                assert covered == [1] * len(units) and total == 148, (nc, lay)   # exact tiling
    # C2 (4 x 2, OS = 2): 76 / 72 / 72 / 76, every unit in exactly two partitions
    lay = _core.partition_layout(4, 74, units)
    assert [s for _, _, s in lay] == [76, 72, 72, 76]

"""Table I coefficient sets of the paper's three desktop testbeds.

Data, not code: PAPER.md:339-358, as bundled by the reference at
/root/reference/pkg/src/sliceplan/testbeds.py:14-60.  They are the parity
fixtures of the partition API; the B200 runtime plans with the measured
profile from ``b200_profile.py`` instead.
"""

from __future__ import annotations

from .costs import HardwareProfile, profile_from_dict


def _doc(name, launch, sigma2, pcie, fp16_gpu, fp16_cpu, int4_gpu, int4_cpu) -> dict:
    def lin(t):
        return {"alpha": t[0], "beta": t[1], "r2": t[2]}

    return {
        "testbed": name,
        "launch": {"alpha": launch, "sigma2": sigma2},
        "pcie": lin(pcie),
        "gemm": {
            "fp16": {"gpu": lin(fp16_gpu), "cpu": lin(fp16_cpu)},
            "int4": {"gpu": lin(int4_gpu), "cpu": lin(int4_cpu)},
        },
    }


#                 launch  sigma2   pcie (a, b, r2)            fp16 gpu                  fp16 cpu
#                 int4 gpu                 int4 cpu
TESTBED_A = _doc("testbed-a", 4.4e-5, 3.4e-6, (3.0e-6, 2.6e-11, 0.985),
                 (1.0e-7, 3.2e-12, 0.997), (7.4e-7, 1.6e-11, 0.988),
                 (4.7e-6, 8.1e-13, 0.999), (1.1e-5, 5.4e-12, 0.998))
TESTBED_B = _doc("testbed-b", 5.7e-5, 5.9e-6, (5.8e-6, 2.5e-11, 0.994),
                 (1.9e-7, 2.6e-12, 0.997), (3.4e-6, 1.5e-11, 0.995),
                 (4.6e-6, 6.5e-13, 0.996), (1.3e-5, 6.5e-12, 0.998))
TESTBED_C = _doc("testbed-c", 5.2e-5, 6.0e-6, (3.7e-6, 4.1e-11, 0.999),
                 (1.4e-7, 3.6e-12, 0.988), (1.8e-6, 2.5e-11, 0.993),
                 (6.4e-6, 9.2e-13, 0.989), (5.6e-7, 8.4e-12, 0.992))

ALL_TESTBEDS: dict[str, dict] = {"a": TESTBED_A, "b": TESTBED_B, "c": TESTBED_C}


def testbed_a() -> HardwareProfile:
    return profile_from_dict(TESTBED_A)


def testbed_b() -> HardwareProfile:
    return profile_from_dict(TESTBED_B)


def testbed_c() -> HardwareProfile:
    return profile_from_dict(TESTBED_C)

"""Seeded randomised parity against the reference build (tests/parity_fuzz.py): 120 cases
over every entry point, edge sizes (1 .. 513, tile and row-group boundaries), real and
complex, dense and CSR. tools/parity_sweep.py runs the long sweep
(profiles/r02_parity_sweep.txt)."""
import pytest

from parity_fuzz import run_case, run_case_cpp, run_case_ext

pytestmark = pytest.mark.gpu


# 100230: a 1 x 1 CSR with no entries times a complex vector -- the case that found the
# unallocated interleaved gather buffer of the complex CSR matvec (a real Delta meeting a
# complex x), fixed in the same round
@pytest.mark.parametrize("seed", list(range(1000, 1120)) + [100230])
def test_random_case_matches_the_reference(ref_arm, seed):
    run_case(seed, ref_arm)


@pytest.mark.parametrize("seed", range(5000, 5080))
def test_random_extended_case_matches_the_reference(ref_arm, seed):
    """Warm starts, the max-abs stop rule, the Ozaki product, 2-3 in-process ranks, and
    couplings that diverge or run out of iterations (status parity)."""
    run_case_ext(seed, ref_arm)


@pytest.mark.parametrize("seed", range(9000, 9060))
def test_random_case_through_the_cpp_dropin(ref_arm, seed):
    """The C++ drop-in entry points on ComplexMatrix carriers (tests/cpp/cpp_api_shim.cpp):
    bitwise the Python mirror's device results, within tolerance of the reference build;
    including several in-process ranks (ipt::b200::set_devices) and repeated solve_single
    calls on one Partition (device-resident problem)."""
    run_case_cpp(seed, ref_arm)

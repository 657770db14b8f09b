"""the reference-side adapter (include/gbnr_gridbatch.hpp)
compiled against the reference's own headers (/root/reference/proj/include, in
place, the oracle/Makefile `ref` recipe) and linked with libgbnr.so.

The program parses a case with the reference's parser, builds its Ybus and
ProfileBatch with the reference's functions, creates a gbnr plan through the
adapter and prints the plan's counters.  On this CPU-only container the plan is
host-only (device -1), so the solve must come back as the reference's
ConfigError (no CPU fallback); with a GPU (device 0) the same program solves and
prints the per-task statuses.  Skipped where /root/reference is absent (the GPU
box).
"""
import os
import subprocess

import numpy as np
import pytest

import util
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case

REF_INC = "/root/reference/proj/include"
JSONDIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"

PROG = r"""
#include <cstdio>
#include <cstdlib>
#include "gbnr_gridbatch.hpp"
#include "gridbatch/case_io.hpp"
using namespace gridbatch;
int main(int argc, char** argv) {
    const GridCase gc = load_case(argv[1]);
    const int device = std::atoi(argv[2]);
    const index_t T = 8;
    const ProfileBatch pb = assemble_profiles(gc, case_scenario(gc, T));
    GbnrSymbolic sym(gc, pb, NrConfig{}, device);
    int64_t st[16];
    if (gbnr_plan_stats(sym.plan(), st) != GBNR_OK) return 2;
    std::printf("stats");
    for (int i = 0; i < 16; ++i) std::printf(" %lld", (long long)st[i]);
    std::printf("\n");
    try {
        const auto res = nr_solve_batch_gbnr(sym, pb);
        std::printf("solved");
        for (const auto& r : res) std::printf(" %d:%d", int(r.status), r.iterations);
        std::printf("\n");
    } catch (const ConfigError& e) {
        std::printf("ConfigError %s\n", e.what());
    }
    return 0;
}
"""


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
@pytest.mark.parametrize("name", ["case14", "synth300"])
def test_adapter_compiles_against_reference_and_runs(name, tmp_path):
    src = tmp_path / "adapter_main.cpp"
    src.write_text(PROG)
    exe = tmp_path / "adapter_main"
    libdir = os.path.join(util.ROOT, "paper_2101_02270_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", f"-I{os.path.join(util.ROOT, 'include')}",
                    f"-I{REF_INC}", f"-I{JSONDIR}", str(src), "-o", str(exe), f"-L{libdir}", "-lgbnr",
                    f"-Wl,-rpath,{libdir}"], check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe), util.case_path(name), "-1"], check=True, capture_output=True,
                         text=True).stdout.splitlines()
    stats = np.array(out[0].split()[1:], dtype=np.int64)
    gc = load_case(util.case_path(name))
    plan = S.NrPlan.from_case(gc, device=-1)
    # the reference's build_ybus / assemble_profiles feed the same symbolic analysis
    assert stats.tolist() == [plan.stats()[k] for k in S.STAT_KEYS]
    assert out[1].startswith("ConfigError")  # host-only plan: no CPU fallback

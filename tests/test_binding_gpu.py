"""The reference-side C++ binding on the GPU: ccsim::NvrarB200Allreduce<T>
(integration/ccsim_nvrar_b200.hpp, the drop-in for NvrarAllreduce<T>,
nvrar.hpp:41-250) runs real all-reduces — run() on device spans, run_host()
on the reference's host spans — in separate rank processes on cuda:0, each
result compared bit for bit with the reference's own oracle
(tests/oracles.hpp nvrar_order_sum) inside the program. The program is
compiled in the build container against the reference headers
(oracle/Makefile `ref`, oracle/binding_check.cpp) and travels prebuilt."""
import os
import subprocess
import tempfile

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "binding_check")


@pytest.mark.parametrize("nodes,gpus", [(2, 1), (1, 2), (2, 2)])
def test_cpp_binding_runs_allreduces(nodes, gpus):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/binding_check not built (needs /root/reference at build time)")
    world = nodes * gpus
    with tempfile.TemporaryDirectory(prefix="nvrar_bind_") as d:
        procs = [subprocess.Popen([EXE, d, str(r), str(nodes), str(gpus), "0"],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for r in range(world)]
        outs = []
        try:
            for p in procs:
                outs.append(p.communicate(timeout=300)[0])
        finally:
            for p in procs:
                if p.poll() is None:
                    p.kill()
                    p.wait()
    text = "".join(outs)
    assert all(p.returncode == 0 for p in procs), text[-4000:]
    assert text.count(": OK") == world, text[-4000:]

"""The reference-side binding (integration/ccsim_nvrar_b200.hpp) compiles
against the reference's own headers and links against libnvrar_b200.so.
CPU only: nothing is launched; the program exercises the host-side error path
(InvalidTopologyError before any device call)."""
import os
import shutil
import subprocess

import pytest

from paper_2511_09557_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"

PROGRAM = r'''
#include <cstdio>
#include "ccsim_nvrar_b200.hpp"
// every drop-in entry point must compile against the reference headers
template <class T>
void uses(ccsim::NvrarB200Allreduce<T>& c) {
  std::span<const T> in;
  std::span<T> out;
  std::span<const std::uint64_t> pk;
  std::span<std::uint64_t> po;
  c.run(in, out, ccsim::NvrarConfig{}, nullptr);
  c.run_host(in, out, ccsim::NvrarConfig{}, nullptr);
  c.rd_inter(pk, po, ccsim::NvrarConfig{}, nullptr);
  c.reduce_scatter(in, out, nullptr);
  c.all_gather(in, out, nullptr);
  c.run_ring(in, out, nullptr);
  c.run_tree(in, out, nullptr);
}
template void uses<float>(ccsim::NvrarB200Allreduce<float>&);
template void uses<std::int32_t>(ccsim::NvrarB200Allreduce<std::int32_t>&);

int main() {
  try {
    ccsim::NvrarB200Allreduce<float> bad(ccsim::ClusterTopology{3, 1}, 0, 0, 1024, nullptr,
                                         nullptr);
  } catch (const ccsim::InvalidTopologyError& e) {
    std::printf("InvalidTopologyError: %s\n", e.what());
    try {
      ccsim::B200RingAllreduce<float> r(ccsim::ClusterTopology{3, 1}, 0, 0, 1024, nullptr,
                                        nullptr);
    } catch (const ccsim::InvalidTopologyError&) {
      try {
        ccsim::B200TreeAllreduce<std::int32_t> t(ccsim::ClusterTopology{6, 1}, 0, 0, 1024,
                                                 nullptr, nullptr);
      } catch (const ccsim::InvalidTopologyError&) {
        return 0;
      }
    }
  }
  return 1;
}
'''


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_binding_compiles_and_maps_errors(tmp_path):
    L.load()
    src = tmp_path / "t.cpp"
    src.write_text(PROGRAM)
    exe = tmp_path / "t"
    libdir = os.path.dirname(L.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O1", f"-I{REF_INC}", f"-I{ROOT}/include",
           f"-I{ROOT}/integration", str(src), "-o", str(exe), f"-L{libdir}", "-l:libnvrar_b200.so",
           f"-Wl,-rpath,{libdir}", "-pthread"]
    subprocess.check_call(cmd)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "power of two" in out.stdout

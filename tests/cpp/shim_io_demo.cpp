// shim_io_demo.cpp — FKF1/FKS1 snapshot round trips through the C++ shim (field_io.hpp:18-135),
// mirroring proj/tests/test_cli_io.cpp:61-100; host only (no GPU needed).  Writes the files
// given on the command line so the Python reader can check the byte layout.
#include <cstdio>
#include <stdexcept>

#include "fastkf_b200.hpp"

int main(int argc, char** argv) {
    using namespace fastkf;
    if (argc < 3) return 2;
    const std::string fpath = argv[1], spath = argv[2];
    Vector data(12 * 7);
    for (Index i = 0; i < data.size(); ++i) data[i] = 0.25 * double(i) - 3.0 + 1e-3 * double(i * i);
    write_field(fpath, 12, 7, data);
    const Field back = read_field(fpath);
    if (back.nx != 12 || back.ny != 7 || back.data.v != data.v) return 3;
    LowRankState st = LowRankState::zero_start(20);
    st.alpha = 3.0;
    st.step = 3;
    st.d = Vector(4);
    for (int i = 0; i < 4; ++i) st.d[i] = 0.1 + 0.2 * i;
    for (Index i = 0; i < 20; ++i) st.mean[i] = 0.5 * double(i) - 1.0;
    Matrix w(20, 4);
    for (Index j = 0; j < 4; ++j)
        for (Index i = 0; i < 20; ++i) w(i, j) = double(i + 1) / double(j + 2);
    write_state(spath, st, w);
    const LowRankState rb = read_state(spath);
    if (rb.alpha != 3.0 || rb.step != 3 || rb.mean.v != st.mean.v || rb.d.v != st.d.v || rb.w.get().a != w.a) return 4;
    int errors = 0;
    try { read_field(spath); } catch (const std::runtime_error&) { ++errors; }          // wrong magic
    try { read_field(fpath + ".missing"); } catch (const std::runtime_error&) { ++errors; }
    try { write_field(fpath, 3, 3, Vector(5)); } catch (const std::invalid_argument&) { ++errors; }
    if (errors != 3) return 5;
    std::printf("io ok\n");
    return 0;
}

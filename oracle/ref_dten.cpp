// ref_dten.cpp — .dten golden files written BY THE REFERENCE'S OWN
// tensor_io.hpp (Eigen-free; compiled in place by oracle/Makefile target
// `dten-goldens`, binary in oracle/_ref/).  Test infrastructure only: the
// engine's streaming reader/writer (csrc/dten_io.cu) and the host mirror
// (paper_2010_10131_b200/tensor_io.py) must read these and write
// byte-identical files.  Usage: ref_dten <out_dir>
#include <string>

#include "atucker/tensor.hpp"
#include "atucker/tensor_io.hpp"

using namespace atucker;

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    write_dten(dir + "/ref_normal_4x3x5_seed7.dten", random_tensor({4, 3, 5}, 7, Distribution::StandardNormal));
    write_dten(dir + "/ref_uniform_6x5x4x3_seed11.dten", random_tensor({6, 5, 4, 3}, 11, Distribution::Uniform01));
    write_dten(dir + "/ref_vec5.dten", DenseTensor({5}, {1, 2, 3, 4, 5}));
    write_dten(dir + "/ref_matrix_3x2.dten", DenseMatrix(3, 2, {1.5, -2.0, 0.25, 4.0, -8.5, 16.0}));
    return 0;
}

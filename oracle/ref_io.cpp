// TEST INFRASTRUCTURE ONLY: `ref_io in.txt out.txt` reads a matrix with the
// reference's read_matrix_file and writes it back with write_matrix_file
// (proj/src/io.cpp, compiled in place); exit status 0, 9 on IoError, 10 else.
#include <cstdio>
#include <exception>

#include "mpsvd/io.hpp"
#include "mpsvd/types.hpp"

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: ref_io in.txt out.txt\n");
    return 1;
  }
  try {
    const mpsvd::DenseMatrix a = mpsvd::read_matrix_file(argv[1]);
    mpsvd::write_matrix_file(argv[2], a);
    return 0;
  } catch (const mpsvd::IoError& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 9;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 10;
  }
}

// Runs the reference-side dispatch (cur_dispatch.cpp) on an m x n matrix read
// from a binary file (int64 m, n, k, loops, r; m*n doubles column-major; k
// int64 initial rows) and prints "I ...", "J ...", "r ..." lines.
#include <cstdio>
#include <fstream>
#include <iostream>

#include "ref_shim.hpp"

namespace slra {
std::pair<CurDecomposition, CaTrace> cross_approx(const EntryOracle& M, Index r, Index k, Index l,
                                                  IndexSet init_rows, int loops, double h);
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  std::ifstream f(argv[1], std::ios::binary);
  int64_t hdr[5];
  f.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
  const int64_t m = hdr[0], n = hdr[1], k = hdr[2], loops = hdr[3], r = hdr[4];
  slra::Matrix A(m, n);
  f.read(reinterpret_cast<char*>(A.data()), 8 * m * n);
  std::vector<slra::Index> init(k);
  f.read(reinterpret_cast<char*>(init.data()), 8 * k);
  try {
    slra::DenseOracle o(A);
    auto [c, trace] = slra::cross_approx(o, r, k, k, slra::IndexSet(init, m), (int)loops, 1.1);
    std::cout << "I";
    for (auto i : c.row_set.indices()) std::cout << ' ' << i;
    std::cout << "\nJ";
    for (auto j : c.col_set.indices()) std::cout << ' ' << j;
    std::cout << "\nr " << c.r << "\nsteps " << trace.steps.size() << "\n";
  } catch (const std::exception& e) {
    std::cout << "error " << e.what() << "\n";
    return 3;
  }
  return 0;
}

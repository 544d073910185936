// Stand-alone driver over the REFERENCE's read_matrix_market_file
// (matrix_market.cpp:22-62). TEST INFRASTRUCTURE ONLY: tests/golden/make_mm.py
// runs it in a subprocess (the reference library carries its own static
// libstdc++, whose iostreams cannot share a process with another copy).
// Usage: ref_mm <in.mtx> <out.bin>; out = int64 code (nnz, or -12 IoError /
// -1 ContractViolation), then n_rows, n_cols, row_ptr, col_idx (int64), values.
#include <cstdint>
#include <cstdio>

extern "C" int64_t ref_mm_read(const char* path, int64_t* n_rows, int64_t* n_cols, int64_t* rp, int64_t* ci,
                               double* v);

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  int64_t nr = 0, nc = 0;
  const int64_t nnz = ref_mm_read(argv[1], &nr, &nc, nullptr, nullptr, nullptr);
  FILE* f = std::fopen(argv[2], "wb");
  if (!f) return 3;
  std::fwrite(&nnz, 8, 1, f);
  if (nnz >= 0) {
    int64_t* rp = new int64_t[nr + 1];
    int64_t* ci = new int64_t[nnz + 1];
    double* v = new double[nnz + 1];
    ref_mm_read(argv[1], &nr, &nc, rp, ci, v);
    std::fwrite(&nr, 8, 1, f);
    std::fwrite(&nc, 8, 1, f);
    std::fwrite(rp, 8, nr + 1, f);
    std::fwrite(ci, 8, nnz, f);
    std::fwrite(v, 8, nnz, f);
  }
  std::fclose(f);
  return 0;
}

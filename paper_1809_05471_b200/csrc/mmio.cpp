// MatrixMarket export of an assembled CSR matrix:
// coordinate format, 1-based indices, `real general`, 17 significant digits.
// Host code: rows are formatted in parallel chunks (OpenMP) and written in
// order, so a C3-sized matrix (95M entries) takes seconds, not minutes.
#include <omp.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/igs_capi.h"

namespace igs {
void set_error(const std::string& msg);
}

extern "C" igs_status igs_write_matrix_market(const char* path, int64_t nrows, int64_t ncols,
                                              const int64_t* indptr, const int64_t* indices,
                                              const double* values) {
  if (!path || nrows < 0 || ncols < 0 || !indptr || (indptr[nrows] > 0 && (!indices || !values))) {
    igs::set_error("bad MatrixMarket arguments");
    return IGS_EARG;
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    igs::set_error(std::string("cannot open ") + path);
    return IGS_EARG;
  }
  const int64_t nnz = indptr[nrows];
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)nrows,
               (long long)ncols, (long long)nnz);
  const int64_t chunk_rows = 4096;
  const int64_t nchunks = (nrows + chunk_rows - 1) / chunk_rows;
  const int64_t batch = 64;  // chunks formatted in parallel, then written in order
  std::vector<std::string> bufs(batch);
  bool ok = true;
  for (int64_t c0 = 0; c0 < nchunks && ok; c0 += batch) {
    const int64_t c1 = c0 + batch < nchunks ? c0 + batch : nchunks;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = c0; c < c1; ++c) {
      std::string& out = bufs[c - c0];
      out.clear();
      char line[96];
      const int64_t r0 = c * chunk_rows, r1 = r0 + chunk_rows < nrows ? r0 + chunk_rows : nrows;
      for (int64_t r = r0; r < r1; ++r)
        for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k) {
          int n = std::snprintf(line, sizeof(line), "%lld %lld %.17g\n", (long long)(r + 1),
                                (long long)(indices[k] + 1), values[k]);
          out.append(line, (size_t)n);
        }
    }
    for (int64_t c = c0; c < c1 && ok; ++c)
      ok = std::fwrite(bufs[c - c0].data(), 1, bufs[c - c0].size(), f) == bufs[c - c0].size();
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    igs::set_error("write failed");
    return IGS_EARG;
  }
  return IGS_OK;
}

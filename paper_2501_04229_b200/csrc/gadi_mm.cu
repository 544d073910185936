// gadi_mm.cu — MatrixMarket ingest (matrix_market.cpp:22-86): the on-disk
// format callers feed the solver through (`mm:path=`, gadi_cli.cpp:65-73).
//
// The banner / size line / entry list are parsed on the host (text); the
// SparseMatrix::from_triplets assembly (sparse.cpp:36-58) -- the
// O(nnz log nnz) part that does not fit host RAM at the BASELINE scales --
// runs on the device: (row, col) keys radix-sorted (stable, CUB), runs of equal
// keys summed left to right in file order, heads compacted by a scan, row
// counts scanned into row_ptr. The reference sums duplicates in std::sort
// order, which is unspecified among equal keys; for duplicate-free files (and
// duplicates whose sum is exact) the result is the reference's bit for bit.
#include <cub/device/device_radix_sort.cuh>
#include <atomic>
#include <charconv>
#include <iterator>
#include <thread>
#include <cctype>
#include <cinttypes>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "gadi_host.cuh"

using namespace gadi_host;

struct gadi_csr {
  int64_t n_rows = 0, n_cols = 0;
  std::vector<int64_t> rp, ci;
  std::vector<double> v;
};

namespace {

std::string lower(std::string s) {
  for (char& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

__global__ void k_mm_keys(const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t m, int64_t ncols,
                          unsigned long long* __restrict__ key, int64_t* __restrict__ idx) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  key[t] = (unsigned long long)r[t] * (unsigned long long)ncols + (unsigned long long)c[t];
  idx[t] = t;
}

// head[t] = 1 when sorted entry t starts a run of equal keys
__global__ void k_mm_heads(const unsigned long long* __restrict__ key, int64_t m, int64_t* __restrict__ head) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  head[t] = (t == 0 || key[t] != key[t - 1]) ? 1 : 0;
}

// one thread per run: sum = x0; sum += x1; ... (sparse.cpp:46-49) in sorted
// (= file, the radix sort being stable) order; write the compacted entry
__global__ void k_mm_sum(const unsigned long long* __restrict__ key, const int64_t* __restrict__ idx,
                         const double* __restrict__ val, const int64_t* __restrict__ pos, int64_t m, int64_t ncols,
                         int64_t* __restrict__ ci, double* __restrict__ v, unsigned long long* __restrict__ rowcnt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m || (t > 0 && key[t] == key[t - 1])) return;
  double sum = val[idx[t]];
  for (int64_t u = t + 1; u < m && key[u] == key[t]; ++u) sum = __dadd_rn(sum, val[idx[u]]);
  const int64_t o = pos[t];  // exclusive scan of heads
  const unsigned long long k = key[t];
  ci[o] = (int64_t)(k % (unsigned long long)ncols);
  v[o] = sum;
  atomicAdd(rowcnt + (int64_t)(k / (unsigned long long)ncols) + 1, 1ull);
}

void assemble(gadi_csr* out, std::vector<int64_t>& r, std::vector<int64_t>& c, std::vector<double>& x,
              int device) {
  const int64_t m = (int64_t)r.size(), nr = out->n_rows, nc = out->n_cols;
  out->rp.assign(nr + 1, 0);
  if (m == 0) return;
  CK(cudaSetDevice(device));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<void*> owned;
  auto al = [&](size_t bytes) {
    void* p = nullptr;
    CK(cudaMallocAsync(&p, std::max<size_t>(bytes, 8), s));
    owned.push_back(p);
    return p;
  };
  try {
    auto* dr = (int64_t*)al(m * 8);
    auto* dc = (int64_t*)al(m * 8);
    auto* dx = (double*)al(m * 8);
    CK(cudaMemcpyAsync(dr, r.data(), m * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dc, c.data(), m * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dx, x.data(), m * 8, cudaMemcpyHostToDevice, s));
    auto* key = (unsigned long long*)al(m * 8);
    auto* key2 = (unsigned long long*)al(m * 8);
    auto* idx = (int64_t*)al(m * 8);
    auto* idx2 = (int64_t*)al(m * 8);
    const unsigned g = (unsigned)((m + 255) / 256);
    k_mm_keys<<<g, 256, 0, s>>>(dr, dc, m, nc, key, idx);
    CKL();
    int bits = 1;
    while (bits < 64 && ((unsigned long long)1 << bits) <= (unsigned long long)nr * (unsigned long long)nc) ++bits;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, m, 0, bits, s));
    void* tmp = al(tb);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, idx2, m, 0, bits, s));
    auto* head = (int64_t*)al((m + 1) * 8);
    auto* pos = (int64_t*)al((m + 1) * 8);
    k_mm_heads<<<g, 256, 0, s>>>(key2, m, head);
    CK(cudaMemsetAsync(head + m, 0, 8, s));
    scan_i64(s, head, pos, m + 1);
    int64_t nnz = 0;
    CK(cudaMemcpyAsync(&nnz, pos + m, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    auto* ci = (int64_t*)al(nnz * 8);
    auto* v = (double*)al(nnz * 8);
    auto* cnt = (unsigned long long*)al((nr + 1) * 8);
    auto* rp = (int64_t*)al((nr + 1) * 8);
    CK(cudaMemsetAsync(cnt, 0, (nr + 1) * 8, s));
    k_mm_sum<<<g, 256, 0, s>>>(key2, idx2, dx, pos, m, nc, ci, v, cnt);
    CKL();
    // row_ptr = inclusive scan of [0, count(row 0), count(row 1), ...]
    size_t sb = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, sb, (const int64_t*)cnt, rp, nr + 1, s));
    void* stmp = al(sb);
    CK(cub::DeviceScan::InclusiveSum(stmp, sb, (const int64_t*)cnt, rp, nr + 1, s));
    out->ci.resize(nnz);
    out->v.resize(nnz);
    CK(cudaMemcpyAsync(out->ci.data(), ci, nnz * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->v.data(), v, nnz * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->rp.data(), rp, (nr + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  } catch (...) {
    for (void* p : owned) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    throw;
  }
  for (void* p : owned) cudaFreeAsync(p, s);
  CK(cudaStreamSynchronize(s));
  CK(cudaStreamDestroy(s));
}

bool is_ws(char ch) { return ch == ' ' || ch == '\n' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f'; }

// The first 3*entries whitespace-separated tokens of buf as (i, j, v) triples,
// parsed by threads over whitespace-aligned chunks (std::from_chars: the
// correctly rounded decimal conversion, as the stream's strtod). Returns 1 on
// success, -1 if there are fewer tokens (truncated), 0 when some token is not
// a plain decimal (then the caller re-parses with the reference's stream loop).
int fast_entries(const std::string& buf, int64_t entries, std::vector<int64_t>& fi, std::vector<int64_t>& fj,
                 std::vector<double>& fv) {
  const size_t n = buf.size();
  const int64_t need = 3 * entries;
  const int T = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<size_t> cut(T + 1, n);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    size_t p = std::max(cut[t - 1], n * t / T);
    while (p < n && !is_ws(buf[p])) ++p;
    cut[t] = p;
  }
  std::vector<int64_t> cnt(T + 1, 0);
  auto tokens = [&](int t, auto&& f) {
    size_t p = cut[t];
    const size_t e = cut[t + 1];
    while (p < e) {
      while (p < e && is_ws(buf[p])) ++p;
      if (p >= e) break;
      size_t q = p;
      while (q < e && !is_ws(buf[q])) ++q;
      if (!f(p, q)) return;
      p = q;
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] { tokens(t, [&](size_t, size_t) { ++cnt[t + 1]; return true; }); });
  for (auto& h : th) h.join();
  th.clear();
  for (int t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
  if (cnt[T] < need) return -1;
  fi.resize(entries);
  fj.resize(entries);
  fv.resize(entries);
  std::atomic<bool> ok{true};
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      int64_t k = cnt[t];
      tokens(t, [&](size_t p, size_t q) {
        if (k >= need || !ok) return false;
        const char* a = buf.data() + p;
        const char* b = buf.data() + q;
        const int64_t e = k / 3;
        if (k % 3 < 2) {  // an index: digits with an optional '-'
          int64_t v = 0;
          auto r = std::from_chars(a, b, v);
          if (r.ec != std::errc() || r.ptr != b) ok = false;
          (k % 3 == 0 ? fi : fj)[e] = v;
        } else {  // a value: [-]digits[.digits][e[+-]digits]
          for (const char* z = a; z < b; ++z)
            if (!((*z >= '0' && *z <= '9') || *z == '-' || *z == '+' || *z == '.' || *z == 'e' || *z == 'E'))
              ok = false;
          double v = 0.0;
          auto r = std::from_chars(a, b, v);
          if (r.ec != std::errc() || r.ptr != b) ok = false;
          fv[e] = v;
        }
        ++k;
        return true;
      });
    });
  for (auto& h : th) h.join();
  return ok ? 1 : 0;
}

}  // namespace

extern "C" {

int gadi_mm_read(const char* path, int32_t device, gadi_csr** out) {
  try {
    if (!path || !out) throw Err(GADI_E_CONTRACT, "mm_read: null argument");
    *out = nullptr;
    std::ifstream in(path);
    if (!in) throw Err(GADI_E_IO, std::string("cannot open ") + path);
    // read_matrix_market, matrix_market.cpp:22-62
    std::string line;
    if (!std::getline(in, line)) throw Err(GADI_E_IO, "matrix market: empty stream");
    std::istringstream hdr(line);
    std::string banner, object, fmt, field, symmetry;
    hdr >> banner >> object >> fmt >> field >> symmetry;
    if (banner != "%%MatrixMarket" || lower(object) != "matrix") throw Err(GADI_E_IO, "matrix market: bad banner");
    if (lower(fmt) != "coordinate") throw Err(GADI_E_IO, "matrix market: only coordinate format supported");
    field = lower(field);
    symmetry = lower(symmetry);
    if (field != "real" && field != "integer") throw Err(GADI_E_IO, "matrix market: only real matrices supported");
    const bool sym = symmetry == "symmetric", skew = symmetry == "skew-symmetric";
    if (!sym && !skew && symmetry != "general")
      throw Err(GADI_E_IO, "matrix market: unsupported symmetry: " + symmetry);
    while (std::getline(in, line))
      if (!line.empty() && line[0] != '%') break;
    std::istringstream dims(line);
    int64_t rows = 0, cols = 0, entries = 0;
    if (!(dims >> rows >> cols >> entries)) throw Err(GADI_E_IO, "matrix market: bad size line");
    if (rows < 0 || cols < 0 || entries < 0) throw Err(GADI_E_CONTRACT, "negative dimension");
    std::vector<int64_t> r, c;
    std::vector<double> x;
    bool bad = false;
    const size_t cap = (size_t)entries * ((sym || skew) ? 2 : 1);
    r.reserve(cap);
    c.reserve(cap);
    x.reserve(cap);
    // the entry list: parsed in parallel when every token is a plain decimal
    // (what write_matrix_market produces), else by the reference's stream loop
    std::string rest((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::vector<int64_t> fi, fj;
    std::vector<double> fv;
    const int fast = fast_entries(rest, entries, fi, fj, fv);
    if (fast < 0) throw Err(GADI_E_IO, "matrix market: truncated entry list");
    std::istringstream slow(fast == 0 ? rest : std::string());
    for (int64_t k = 0; k < entries; ++k) {
      int64_t i = 0, j = 0;
      double v = 0.0;
      if (fast) {
        i = fi[k];
        j = fj[k];
        v = fv[k];
      } else if (!(slow >> i >> j >> v)) {
        throw Err(GADI_E_IO, "matrix market: truncated entry list");
      }
      --i;
      --j;  // 1-based on disk
      if (i < 0 || i >= rows || j < 0 || j >= cols) bad = true;  // from_triplets throws after parsing
      r.push_back(i);
      c.push_back(j);
      x.push_back(v);
      if (i != j && (sym || skew)) {
        if (j >= rows || i >= cols) bad = true;
        r.push_back(j);
        c.push_back(i);
        x.push_back(skew ? -v : v);
      }
    }
    if (bad) throw Err(GADI_E_CONTRACT, "triplet out of range");  // sparse.cpp:50
    std::unique_ptr<gadi_csr> m(new gadi_csr);
    m->n_rows = rows;
    m->n_cols = cols;
    assemble(m.get(), r, c, x, device);
    *out = m.release();
  } catch (const Err& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return GADI_E_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GADI_E_CUDA;
  }
  return GADI_OK;
}

int gadi_csr_view(const gadi_csr* m, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, const int64_t** row_ptr,
                  const int64_t** col_idx, const double** values) {
  if (!m) return GADI_E_CONTRACT;
  if (n_rows) *n_rows = m->n_rows;
  if (n_cols) *n_cols = m->n_cols;
  if (nnz) *nnz = (int64_t)m->v.size();
  if (row_ptr) *row_ptr = m->rp.data();
  if (col_idx) *col_idx = m->ci.data();
  if (values) *values = m->v.data();
  return GADI_OK;
}

int gadi_csr_destroy(gadi_csr* m) {
  delete m;
  return GADI_OK;
}

// write_matrix_market (matrix_market.cpp:64-86): "symmetric" (lower triangle)
// when A equals its transpose exactly, else "general"; %.17g values.
int gadi_mm_write(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_idx,
                  const double* values) {
  try {
    if (!path || !row_ptr || (row_ptr[n_rows] > 0 && (!col_idx || !values)))
      throw Err(GADI_E_CONTRACT, "mm_write: null argument");
    const int64_t nnz = row_ptr[n_rows];
    // is_symmetric (sparse.cpp:128-132): square, and the transpose has the same arrays
    bool symmetric = n_rows == n_cols;
    if (symmetric) {
      std::vector<int64_t> trp(n_cols + 1, 0), tci(nnz);
      std::vector<double> tv(nnz);
      for (int64_t k = 0; k < nnz; ++k) ++trp[col_idx[k] + 1];
      for (int64_t j = 0; j < n_cols; ++j) trp[j + 1] += trp[j];
      std::vector<int64_t> next(trp.begin(), trp.end() - 1);
      for (int64_t i = 0; i < n_rows; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          const int64_t p = next[col_idx[k]]++;
          tci[p] = i;
          tv[p] = values[k];
        }
      for (int64_t i = 0; i <= n_rows && symmetric; ++i) symmetric = trp[i] == row_ptr[i];
      for (int64_t k = 0; k < nnz && symmetric; ++k) symmetric = tci[k] == col_idx[k] && tv[k] == values[k];
    }
    std::ofstream f(path);
    if (!f) throw Err(GADI_E_IO, std::string("cannot open ") + path + " for writing");
    f << "%%MatrixMarket matrix coordinate real " << (symmetric ? "symmetric" : "general") << "\n";
    int64_t entries = nnz;
    if (symmetric) {
      entries = 0;
      for (int64_t i = 0; i < n_rows; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
          if (col_idx[k] <= i) ++entries;
    }
    f << n_rows << " " << n_cols << " " << entries << "\n";
    char buf[96];
    for (int64_t i = 0; i < n_rows; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        const int64_t j = col_idx[k];
        if (symmetric && j > i) continue;
        std::snprintf(buf, sizeof(buf), "%" PRId64 " %" PRId64 " %.17g\n", i + 1, j + 1, values[k]);
        f << buf;
      }
    if (!f) throw Err(GADI_E_IO, std::string("write failed: ") + path);
  } catch (const Err& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GADI_E_CUDA;
  }
  return GADI_OK;
}

}  // extern "C"

// LIBSVM text ingestion (§8(f) item 3): a parallel parser with the reference's
// exact semantics -- parse_libsvm, proj/src/io.cpp:54-132 -- producing the CSR
// arrays the device upload consumes.
//
// The text is cut into one range per host worker at line boundaries. Each
// worker parses its lines with the reference's per-line rules:
//   * skip_ws, a '+'-tolerant from_chars for the label and the values
//     (io.cpp:22-38);
//   * labels -1 / 0 / +1 (io.cpp:40-45);
//   * 1-based, strictly ascending int32 indices followed by ':'.
// The first offending line in file order is reported with the reference's
// message and 1-based line number.  Blank lines count as lines and are skipped.
//
// The ranges are then stitched together: row offsets rebased, columns and
// values concatenated in place.
// std::from_chars is the same routine the reference uses, so every parsed
// double is bit-identical to the reference's.
#include "ingest.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <system_error>

#include "hostio.h"

namespace tb {

namespace {

struct LineError {
  int kind = 0;  // 0 none, 1 ParseError, 2 UnsupportedLabelError
  std::string what;
  uint64_t local_line = 0;
};

const char* skip_ws(const char* p, const char* end) {
  while (p < end && (*p == ' ' || *p == '\t')) ++p;
  return p;
}

// io.cpp:22-38
bool parse_double(const char*& p, const char* end, const char* what, double* out, LineError* e) {
  const char* start = (p < end && *p == '+') ? p + 1 : p;
  double value;
  auto [next, ec] = std::from_chars(start, end, value);
  if (ec == std::errc::invalid_argument) {
    e->kind = 1;
    e->what = std::string("expected ") + what + " near '" +
              std::string(p, std::min<std::ptrdiff_t>(end - p, 12)) + "'";
    return false;
  }
  if (ec == std::errc::result_out_of_range || !std::isfinite(value)) {
    e->kind = 1;
    e->what = std::string(what) + " is outside the finite double range";
    return false;
  }
  p = next;
  *out = value;
  return true;
}

struct Part {
  const char* begin = nullptr;
  const char* end = nullptr;
  std::vector<int64_t> row_nnz;
  std::vector<int32_t> cols;
  std::vector<double> vals, y;
  uint64_t lines = 0;  // '\n'-terminated lines seen (the error's line is local)
  uint64_t max_index = 0;
  LineError err;
};

// One line (without its '\n'); false on the first error (recorded in P.err).
bool parse_line(const char* ptr, const char* end, Part& P) {
  if (ptr < end && end[-1] == '\r') --end;
  ptr = skip_ws(ptr, end);
  if (ptr == end) return true;  // blank line
  double raw;
  if (!parse_double(ptr, end, "label", &raw, &P.err)) return false;
  if (ptr < end && *ptr != ' ' && *ptr != '\t') {
    P.err = {1, "trailing characters after the label", 0};
    return false;
  }
  double label;  // io.cpp:40-45
  if (raw == 1.0)
    label = 1.0;
  else if (raw == -1.0 || raw == 0.0)
    label = -1.0;
  else {
    P.err = {2, "label " + std::to_string(raw) + " not in {-1, 0, +1}", 0};
    return false;
  }
  P.y.push_back(label);
  int64_t prev_index = 0, count = 0;
  for (;;) {
    ptr = skip_ws(ptr, end);
    if (ptr == end) break;
    int64_t index;
    const char* index_start = (*ptr == '+') ? ptr + 1 : ptr;
    auto [next, ec] = std::from_chars(index_start, end, index);
    if (ec != std::errc()) {
      P.err = {1,
               "expected a feature index near '" +
                   std::string(ptr, std::min<std::ptrdiff_t>(end - ptr, 12)) + "'",
               0};
      return false;
    }
    ptr = next;
    if (ptr == end || *ptr != ':') {
      P.err = {1, "expected ':' after feature index " + std::to_string(index), 0};
      return false;
    }
    ++ptr;
    if (index < 1) {
      P.err = {1, "feature index " + std::to_string(index) + " is not 1-based", 0};
      return false;
    }
    if (index <= prev_index) {
      P.err = {1,
               "feature index " + std::to_string(index) + " not strictly ascending (previous " +
                   std::to_string(prev_index) + ")",
               0};
      return false;
    }
    if (index > std::numeric_limits<int32_t>::max()) {
      P.err = {1, "feature index " + std::to_string(index) + " too large", 0};
      return false;
    }
    double value;
    if (!parse_double(ptr, end, "feature value", &value, &P.err)) return false;
    if (ptr < end && *ptr != ' ' && *ptr != '\t') {
      P.err = {1, "trailing characters after a feature value", 0};
      return false;
    }
    prev_index = index;
    P.cols.push_back(static_cast<int32_t>(index - 1));
    P.vals.push_back(value);
    if (static_cast<uint64_t>(index) > P.max_index) P.max_index = static_cast<uint64_t>(index);
    ++count;
  }
  P.row_nnz.push_back(count);
  return true;
}

// load_dense's per-line rules (io.cpp:171-192): a label, then exactly n values.
bool parse_dense_line(const char* ptr, const char* end, uint64_t n, Part& P) {
  if (ptr < end && end[-1] == '\r') --end;
  ptr = skip_ws(ptr, end);
  if (ptr == end) return true;  // blank line
  double raw;
  if (!parse_double(ptr, end, "label", &raw, &P.err)) return false;
  double label;  // map_label, io.cpp:40-45
  if (raw == 1.0)
    label = 1.0;
  else if (raw == -1.0 || raw == 0.0)
    label = -1.0;
  else {
    P.err = {2, "label " + std::to_string(raw) + " not in {-1, 0, +1}", 0};
    return false;
  }
  P.y.push_back(label);
  uint64_t fields = 0;
  for (;;) {
    ptr = skip_ws(ptr, end);
    if (ptr == end) break;
    if (fields == n) {
      P.err = {1, "more than " + std::to_string(n) + " values", 0};
      return false;
    }
    double v;
    if (!parse_double(ptr, end, "feature value", &v, &P.err)) return false;
    P.vals.push_back(v);
    ++fields;
  }
  if (fields != n) {
    P.err = {1, "expected " + std::to_string(n) + " values, got " + std::to_string(fields), 0};
    return false;
  }
  return true;
}

template <class LineFn>
void parse_part_with(Part& P, LineFn line_fn) {
  const char* p = P.begin;
  while (p < P.end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', P.end - p));
    const char* le = nl ? nl : P.end;
    ++P.lines;
    if (!line_fn(p, le, P)) {
      P.err.local_line = P.lines;
      return;
    }
    p = nl ? nl + 1 : P.end;
  }
}

// Line-boundary ranges of the text, ~4 MB or more each, one or more per worker.
std::vector<Part> split_parts(const char* data, uint64_t len) {
  const size_t want = std::max<size_t>(1, std::min<size_t>((size_t)host_workers() * 4,
                                                           (size_t)(len >> 22) + 1));
  std::vector<const char*> cut{data};
  for (size_t k = 1; k < want; ++k) {
    const char* p = data + len * k / want;
    if (p <= cut.back()) continue;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', data + len - p));
    if (!nl) break;
    if (nl + 1 > cut.back() && nl + 1 < data + len) cut.push_back(nl + 1);
  }
  cut.push_back(data + len);
  std::vector<Part> parts(cut.size() - 1);
  for (size_t k = 0; k + 1 < cut.size(); ++k) {
    parts[k].begin = cut[k];
    parts[k].end = cut[k + 1];
  }
  return parts;
}

// The first error in file order (the lines of earlier ranges are all valid).
void raise_first_error(const std::vector<Part>& parts) {
  uint64_t line_base = 0;
  for (const Part& P : parts) {
    if (P.err.kind) {
      const uint64_t line = line_base + P.err.local_line;
      throw ParseFailure(P.err.kind == 2 ? TRON_ERR_UNSUPPORTED_LABEL : TRON_ERR_PARSE,
                         "line " + std::to_string(line) + ": " + P.err.what, line);
    }
    line_base += P.lines;
  }
}

template <class Fn>
auto with_mapped_file(const char* path, Fn fn) {
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) throw ParseFailure(TRON_ERR_ARGUMENT, std::string("cannot open ") + path, 0);
  struct stat st;
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    throw ParseFailure(TRON_ERR_ARGUMENT, std::string("cannot stat ") + path, 0);
  }
  const size_t len = (size_t)st.st_size;
  if (len == 0) {
    ::close(fd);
    return fn("", (uint64_t)0);
  }
  void* map = ::mmap(nullptr, len, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
  ::close(fd);
  if (map == MAP_FAILED) throw ParseFailure(TRON_ERR_ARGUMENT, std::string("cannot map ") + path, 0);
  try {
    auto out = fn(static_cast<const char*>(map), (uint64_t)len);
    ::munmap(map, len);
    return out;
  } catch (...) {
    ::munmap(map, len);
    throw;
  }
}

void parse_part(Part& P) {
  const char* p = P.begin;
  while (p < P.end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', P.end - p));
    const char* le = nl ? nl : P.end;
    ++P.lines;
    if (!parse_line(p, le, P)) {
      P.err.local_line = P.lines;
      return;
    }
    p = nl ? nl + 1 : P.end;
  }
}

}  // namespace

ParsedProblem parse_libsvm_buffer(const char* data, uint64_t len, uint64_t n_override) {
  std::vector<Part> parts = split_parts(data, len);
  const size_t np = parts.size();
  parallel_for(np, 1, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k) parse_part(parts[k]);
  });
  raise_first_error(parts);
  ParsedProblem out;
  uint64_t rows = 0, nnz = 0, max_index = 0;
  std::vector<uint64_t> row0(np + 1, 0), nz0(np + 1, 0);
  for (size_t k = 0; k < np; ++k) {
    row0[k + 1] = row0[k] + parts[k].y.size();
    nz0[k + 1] = nz0[k] + parts[k].vals.size();
    max_index = std::max(max_index, parts[k].max_index);
  }
  rows = row0[np];
  nnz = nz0[np];
  out.row_offsets.resize(rows + 1);
  out.col_indices.resize(nnz);
  out.values.resize(nnz);
  out.y.resize(rows);
  out.row_offsets[0] = 0;
  parallel_for(np, 1, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k) {
      const Part& P = parts[k];
      int64_t off = (int64_t)nz0[k];
      for (size_t r = 0; r < P.row_nnz.size(); ++r) {
        off += P.row_nnz[r];
        out.row_offsets[row0[k] + r + 1] = off;
      }
      std::memcpy(out.col_indices.data() + nz0[k], P.cols.data(), P.cols.size() * sizeof(int32_t));
      std::memcpy(out.values.data() + nz0[k], P.vals.data(), P.vals.size() * sizeof(double));
      std::memcpy(out.y.data() + row0[k], P.y.data(), P.y.size() * sizeof(double));
    }
  });
  out.cols = max_index;  // io.cpp:120-129
  if (n_override > 0) {
    if (max_index > n_override)
      throw ParseFailure(TRON_ERR_PARSE,
                         "feature index " + std::to_string(max_index) +
                             " exceeds the requested dimension " + std::to_string(n_override),
                         0);
    out.cols = n_override;
  }
  return out;
}

ParsedProblem parse_libsvm_file(const char* path, uint64_t n_override) {
  return with_mapped_file(path, [&](const char* d, uint64_t len) {
    return parse_libsvm_buffer(d, len, n_override);
  });
}

ParsedProblem load_dense_buffer(const char* data, uint64_t len, uint64_t n) {
  std::vector<Part> parts = split_parts(data, len);
  const size_t np = parts.size();
  parallel_for(np, 1, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k)
      parse_part_with(parts[k], [n](const char* a, const char* z, Part& P) {
        return parse_dense_line(a, z, n, P);
      });
  });
  raise_first_error(parts);
  ParsedProblem out;
  out.dense = true;
  out.cols = n;
  std::vector<uint64_t> row0(np + 1, 0);
  for (size_t k = 0; k < np; ++k) row0[k + 1] = row0[k] + parts[k].y.size();
  const uint64_t rows = row0[np];
  out.row_offsets.clear();
  out.values.resize(rows * n);
  out.y.resize(rows);
  parallel_for(np, 1, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k) {
      const Part& P = parts[k];
      std::memcpy(out.values.data() + row0[k] * n, P.vals.data(), P.vals.size() * sizeof(double));
      std::memcpy(out.y.data() + row0[k], P.y.data(), P.y.size() * sizeof(double));
    }
  });
  return out;
}

ParsedProblem load_dense_file(const char* path, uint64_t n) {
  return with_mapped_file(path, [&](const char* d, uint64_t len) { return load_dense_buffer(d, len, n); });
}

// ---- binary cache ---------------------------------------------------------
namespace {
constexpr char kMagic[8] = {'T', 'R', 'O', 'N', 'B', 'I', 'N', '1'};
struct BinHeader {
  char magic[8];
  uint64_t layout;  // 0 CSR, 1 dense
  uint64_t rows, cols, nnz;
};
}  // namespace

void save_binary(const ParsedProblem& p, const char* path) {
  BinHeader h;
  std::memcpy(h.magic, kMagic, sizeof(kMagic));
  h.layout = p.dense ? 1 : 0;
  h.rows = p.y.size();
  h.cols = p.cols;
  h.nnz = p.values.size();
  const std::string tmp = std::string(path) + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) throw ParseFailure(TRON_ERR_ARGUMENT, std::string("cannot create ") + tmp, 0);
  auto put = [&](const void* d, size_t bytes) {
    if (bytes && std::fwrite(d, 1, bytes, f) != bytes) {
      std::fclose(f);
      std::remove(tmp.c_str());
      throw ParseFailure(TRON_ERR_ARGUMENT, std::string("short write to ") + tmp, 0);
    }
  };
  put(&h, sizeof(h));
  if (!p.dense) {
    put(p.row_offsets.data(), p.row_offsets.size() * sizeof(int64_t));
    put(p.col_indices.data(), p.col_indices.size() * sizeof(int32_t));
  }
  put(p.values.data(), p.values.size() * sizeof(double));
  put(p.y.data(), p.y.size() * sizeof(double));
  if (std::fclose(f) != 0 || std::rename(tmp.c_str(), path) != 0)
    throw ParseFailure(TRON_ERR_ARGUMENT, std::string("cannot write ") + path, 0);
}

ParsedProblem load_binary(const char* path) {
  return with_mapped_file(path, [&](const char* d, uint64_t len) {
    BinHeader h;
    if (len < sizeof(h)) throw ParseFailure(TRON_ERR_PARSE, std::string(path) + ": not a TRONBIN1 file", 0);
    std::memcpy(&h, d, sizeof(h));
    if (std::memcmp(h.magic, kMagic, sizeof(kMagic)) != 0 || h.layout > 1)
      throw ParseFailure(TRON_ERR_PARSE, std::string(path) + ": not a TRONBIN1 file", 0);
    ParsedProblem p;
    p.dense = h.layout == 1;
    p.cols = h.cols;
    const uint64_t want = sizeof(h) + (p.dense ? 0 : (h.rows + 1) * 8 + h.nnz * 4) + h.nnz * 8 + h.rows * 8;
    if (len != want || (p.dense && h.nnz != h.rows * h.cols))
      throw ParseFailure(TRON_ERR_PARSE, std::string(path) + ": truncated or inconsistent TRONBIN1 file", 0);
    const char* q = d + sizeof(h);
    auto take = [&](auto& v, uint64_t count) {
      v.resize(count);
      std::memcpy(v.data(), q, count * sizeof(v[0]));
      q += count * sizeof(v[0]);
    };
    if (!p.dense) {
      take(p.row_offsets, h.rows + 1);
      take(p.col_indices, h.nnz);
    } else {
      p.row_offsets.clear();
    }
    take(p.values, h.nnz);
    take(p.y, h.rows);
    return p;
  });
}

}  // namespace tb

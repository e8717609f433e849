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
  // ranges at line boundaries, ~4 MB or more each
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
  const size_t np = cut.size() - 1;
  std::vector<Part> parts(np);
  for (size_t k = 0; k < np; ++k) {
    parts[k].begin = cut[k];
    parts[k].end = cut[k + 1];
  }
  parallel_for(np, 1, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k) parse_part(parts[k]);
  });
  // the first error in file order (lines of earlier ranges are all valid)
  uint64_t line_base = 0;
  for (const Part& P : parts) {
    if (P.err.kind) {
      const uint64_t line = line_base + P.err.local_line;
      throw ParseFailure(P.err.kind == 2 ? TRON_ERR_UNSUPPORTED_LABEL : TRON_ERR_PARSE,
                         "line " + std::to_string(line) + ": " + P.err.what, line);
    }
    line_base += P.lines;
  }
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
    return parse_libsvm_buffer("", 0, n_override);
  }
  void* map = ::mmap(nullptr, len, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
  ::close(fd);
  if (map == MAP_FAILED) throw ParseFailure(TRON_ERR_ARGUMENT, std::string("cannot map ") + path, 0);
  try {
    ParsedProblem p = parse_libsvm_buffer(static_cast<const char*>(map), len, n_override);
    ::munmap(map, len);
    return p;
  } catch (...) {
    ::munmap(map, len);
    throw;
  }
}

}  // namespace tb

// LIBSVM text ingestion with the reference's semantics (io.cpp:54-132).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tron_b200.h"

namespace tb {

struct ParsedProblem {
  bool dense = false;  // dense: values row-major rows x cols, no offsets / indices
  std::vector<int64_t> row_offsets{0};
  std::vector<int32_t> col_indices;
  std::vector<double> values, y;
  uint64_t cols = 0;
};

// ParseError / UnsupportedLabelError (error.hpp:28-43): status + message
// ("line N: ..." when line > 0) + the 1-based line.
struct ParseFailure : std::runtime_error {
  int status;
  uint64_t line;
  ParseFailure(int s, const std::string& m, uint64_t l) : std::runtime_error(m), status(s), line(l) {}
};

ParsedProblem parse_libsvm_buffer(const char* data, uint64_t len, uint64_t n_override);
ParsedProblem parse_libsvm_file(const char* path, uint64_t n_override);
// load_dense (io.cpp:164-197): "label v1 ... vn" per line, exactly n values.
ParsedProblem load_dense_buffer(const char* data, uint64_t len, uint64_t n);
ParsedProblem load_dense_file(const char* path, uint64_t n);
// Binary cache of a parsed problem (little-endian; "TRONBIN1" header, the
// layout, rows, cols, nnz, then the arrays): written once, read back at
// storage speed instead of re-parsing text.
void save_binary(const ParsedProblem& p, const char* path);
ParsedProblem load_binary(const char* path);

}  // namespace tb

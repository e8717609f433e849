// LIBSVM text ingestion with the reference's semantics (io.cpp:54-132).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tron_b200.h"

namespace tb {

struct ParsedProblem {
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

}  // namespace tb

// Ingest / egest formats of the reference (proj/include/eigmod/io.hpp,
// proj/src/io.cpp:59-194): Matrix Market "array real
// symmetric|general" and plain CSV with an optional "# signs:" line.
//
// Same accepted grammar, values and error messages as the reference, built
// for n in the tens of thousands (an n = 32768 Q is ~25 GB of CSV text): the
// file is read in one block, split into lines, and the lines are parsed
// (std::from_chars, correctly rounded) and formatted (std::to_chars with
// precision 17, byte-identical to the reference's "%.17g") by all host
// threads. Errors are reported for the first offending line in file order,
// as the reference's sequential reader does.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "eigmod_b200/eigmod.hpp"

namespace eigmod {

namespace {

std::string lower(std::string s) {
  std::transform(s.begin(), s.end(), s.begin(),
                 [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
  return s;
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n'; }

std::string_view trim(std::string_view s) {
  std::size_t b = 0, e = s.size();
  while (b < e && is_space(s[b])) ++b;
  while (e > b && is_space(s[e - 1])) --e;
  return s.substr(b, e - b);
}

bool parse_double(std::string_view tok, double* out) {
  const char* first = tok.data();
  const char* last = tok.data() + tok.size();
  auto [p, ec] = std::from_chars(first, last, *out);
  return ec == std::errc{} && p == last;
}

[[noreturn]] void bad_token(const std::string& path, std::string_view tok) {
  throw FormatError(path + ": bad numeric token '" + std::string(tok) + "'");
}

std::string read_all(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw FormatError(path + ": cannot open");
  in.seekg(0, std::ios::end);
  const std::streamoff size = in.tellg();
  in.seekg(0, std::ios::beg);
  std::string data(size > 0 ? static_cast<std::size_t>(size) : 0, '\0');
  if (size > 0) in.read(data.data(), size);
  return data;
}

// Line views as std::getline yields them (the final line may lack '\n').
std::vector<std::string_view> split_lines(const std::string& data) {
  std::vector<std::string_view> lines;
  std::size_t pos = 0;
  while (pos < data.size()) {
    const void* nl = std::memchr(data.data() + pos, '\n', data.size() - pos);
    const std::size_t end = nl ? static_cast<const char*>(nl) - data.data() : data.size();
    lines.emplace_back(data.data() + pos, end - pos);
    pos = end + 1;
  }
  return lines;
}

std::size_t format_value(char* buf, double v) {
  auto r = std::to_chars(buf, buf + 40, v, std::chars_format::general, 17);
  return static_cast<std::size_t>(r.ptr - buf);
}

struct FileCloser {
  void operator()(std::FILE* f) const {
    if (f) std::fclose(f);
  }
};
using FilePtr = std::unique_ptr<std::FILE, FileCloser>;

FilePtr open_for_write(const std::string& path) {
  FilePtr f(std::fopen(path.c_str(), "w"));
  if (!f) throw FormatError(path + ": cannot open for writing");
  return f;
}

// Formats items [0, count) with emit(i, buffer) in parallel chunks and writes
// the chunks in order.
template <class Emit>
void parallel_write(std::FILE* f, std::size_t count, std::size_t per_item, Emit&& emit) {
  constexpr std::size_t kChunk = 1 << 14;
  const std::size_t nchunks = (count + kChunk - 1) / kChunk;
  const std::size_t batch = 64;  // chunks formatted per parallel round
  std::vector<std::string> bufs(std::min(nchunks, batch));
  for (std::size_t c0 = 0; c0 < nchunks; c0 += batch) {
    const std::size_t c1 = std::min(nchunks, c0 + batch);
#pragma omp parallel for schedule(dynamic, 1)
    for (std::ptrdiff_t c = static_cast<std::ptrdiff_t>(c0); c < static_cast<std::ptrdiff_t>(c1);
         ++c) {
      std::string& b = bufs[c - c0];
      const std::size_t i0 = c * kChunk, i1 = std::min(count, i0 + kChunk);
      b.resize((i1 - i0) * per_item);
      std::size_t len = 0;
      for (std::size_t i = i0; i < i1; ++i) len += emit(i, b.data() + len);
      b.resize(len);
    }
    for (std::size_t c = c0; c < c1; ++c) std::fwrite(bufs[c - c0].data(), 1, bufs[c - c0].size(), f);
  }
}

}  // namespace

SymmetricDense read_matrix_market(const std::string& path) {
  const std::string data = read_all(path);
  const std::vector<std::string_view> lines = split_lines(data);
  if (lines.empty()) throw FormatError(path + ": empty file");
  std::istringstream hdr{std::string(lines[0])};
  std::string banner, object, format, field, symmetry;
  hdr >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%MatrixMarket" || lower(object) != "matrix" || lower(format) != "array" ||
      lower(field) != "real")
    throw FormatError(path + ": expected '%%MatrixMarket matrix array real symmetric' header");
  const std::string sym = lower(symmetry);
  if (sym != "symmetric" && sym != "general")
    throw FormatError(path + ": unsupported symmetry '" + symmetry + "'");
  // dimension line: the first non-empty, non-comment line (io.cpp:78-81); at
  // EOF the last line read is parsed, as std::getline leaves it in place
  std::size_t li = 1;
  std::string_view dline = lines[0];
  for (; li < lines.size(); ++li) {
    dline = lines[li];
    const std::string_view t = trim(dline);
    if (!t.empty() && t[0] != '%') break;
  }
  std::istringstream dims{std::string(dline)};
  long rows = 0, cols = 0;
  if (!(dims >> rows >> cols) || rows <= 0 || cols <= 0)
    throw FormatError(path + ": bad dimension line");
  if (rows != cols) throw FormatError(path + ": matrix not square");
  const std::size_t n = static_cast<std::size_t>(rows);
  const std::size_t want = (sym == "symmetric") ? n * (n + 1) / 2 : n * n;
  // value lines after the dimension line (comments and blanks skipped)
  std::vector<std::string_view> vals;
  vals.reserve(want);
  for (std::size_t i = li + 1; i < lines.size() && vals.size() < want; ++i) {
    const std::string_view t = trim(lines[i]);
    if (t.empty() || t[0] == '%') continue;
    vals.push_back(t);
  }
  std::vector<double> v(vals.size());
  std::vector<char> ok(vals.size(), 1);
#pragma omp parallel for schedule(static)
  for (std::ptrdiff_t i = 0; i < static_cast<std::ptrdiff_t>(vals.size()); ++i)
    ok[i] = parse_double(vals[i], &v[i]);
  for (std::size_t i = 0; i < vals.size(); ++i)
    if (!ok[i]) bad_token(path, vals[i]);
  if (vals.size() < want) throw FormatError(path + ": truncated data section");
  Matrix m(n, n);
  if (sym == "symmetric") {  // column-major lower triangle
#pragma omp parallel for schedule(dynamic, 16)
    for (std::ptrdiff_t j = 0; j < static_cast<std::ptrdiff_t>(n); ++j) {
      std::size_t idx = static_cast<std::size_t>(j) * n - static_cast<std::size_t>(j) * (j - 1) / 2;
      for (std::size_t i = j; i < n; ++i, ++idx) {
        m(i, j) = v[idx];
        m(j, i) = v[idx];
      }
    }
  } else {
#pragma omp parallel for schedule(static)
    for (std::ptrdiff_t j = 0; j < static_cast<std::ptrdiff_t>(n); ++j)
      for (std::size_t i = 0; i < n; ++i) m(i, j) = v[j * n + i];
  }
  try {
    return SymmetricDense::from(m);
  } catch (const std::invalid_argument& e) {
    throw FormatError(path + ": " + e.what());
  }
}

void write_matrix_market(const std::string& path, const SymmetricDense& a) {
  FilePtr f = open_for_write(path);
  std::fputs("%%MatrixMarket matrix array real symmetric\n", f.get());
  std::fprintf(f.get(), "%zu %zu\n", a.n, a.n);
  // items: columns j, each the lower part i >= j
  const std::size_t n = a.n;
  constexpr std::size_t kPer = 26;
  // columns formatted in parallel batches, written in order
  std::vector<std::string> colbuf;
  const std::size_t batch = 256;
  for (std::size_t j0 = 0; j0 < n; j0 += batch) {
    const std::size_t j1 = std::min(n, j0 + batch);
    colbuf.assign(j1 - j0, std::string());
#pragma omp parallel for schedule(dynamic, 1)
    for (std::ptrdiff_t j = static_cast<std::ptrdiff_t>(j0); j < static_cast<std::ptrdiff_t>(j1);
         ++j) {
      std::string& b = colbuf[j - j0];
      b.resize((n - j) * kPer);
      std::size_t len = 0;
      for (std::size_t i = j; i < n; ++i) {
        len += format_value(b.data() + len, a.entries(i, j));
        b[len++] = '\n';
      }
      b.resize(len);
    }
    for (const auto& b : colbuf) std::fwrite(b.data(), 1, b.size(), f.get());
  }
}

std::vector<int> parse_signs(const std::string& text) {
  std::vector<int> signs;
  std::istringstream ss(text);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    const std::string t(trim(tok));
    if (t == "+1" || t == "1" || t == "+") signs.push_back(1);
    else if (t == "-1" || t == "-") signs.push_back(-1);
    else throw FormatError("bad sign token '" + t + "'");
  }
  if (signs.empty()) throw FormatError("empty sign list");
  return signs;
}

CsvMatrix read_csv_matrix(const std::string& path) {
  const std::string data = read_all(path);
  const std::vector<std::string_view> lines = split_lines(data);
  CsvMatrix out;
  // sequential classification (io.cpp:147-160): the "# signs:" comment counts
  // only as the first non-empty line
  std::vector<std::string_view> rows;
  rows.reserve(lines.size());
  bool first = true;
  for (const std::string_view& l : lines) {
    const std::string_view t = trim(l);
    if (t.empty()) continue;
    if (t[0] == '#') {
      const auto pos = t.find("signs:");
      if (first && pos != std::string_view::npos)
        out.signs = parse_signs(std::string(t.substr(pos + 6)));
      first = false;
      continue;
    }
    first = false;
    rows.push_back(t);
  }
  if (rows.empty()) throw FormatError(path + ": no data rows");
  // per-row parse in parallel; first error in file order wins
  const std::size_t nr = rows.size();
  std::vector<std::size_t> ncol(nr, 0);
  std::vector<std::ptrdiff_t> bad(nr, -1);  // offset of the first bad token
  std::vector<std::size_t> badlen(nr, 0);
  // std::getline(ss, tok, ',') semantics (io.cpp:165-166): a trailing comma
  // ends the row without an empty last token
  auto count_cols = [](std::string_view r) {
    const std::size_t commas = static_cast<std::size_t>(std::count(r.begin(), r.end(), ','));
    return commas + 1 - ((!r.empty() && r.back() == ',') ? 1 : 0);
  };
  const std::size_t width = count_cols(rows[0]);
  Matrix values(nr, width);
#pragma omp parallel for schedule(dynamic, 64)
  for (std::ptrdiff_t i = 0; i < static_cast<std::ptrdiff_t>(nr); ++i) {
    const std::string_view r = rows[i];
    std::size_t c = 0, pos = 0;
    while (true) {
      const std::size_t comma = r.find(',', pos);
      const std::string_view tok = r.substr(pos, comma == std::string_view::npos ? r.npos
                                                                                : comma - pos);
      const std::string_view tt = trim(tok);
      double v = 0.0;
      if (!parse_double(tt, &v)) {
        bad[i] = tt.data() - r.data();
        badlen[i] = tt.size();
        break;
      }
      if (c < width) values(i, c) = v;
      ++c;
      if (comma == std::string_view::npos || comma + 1 == r.size()) break;
      pos = comma + 1;
    }
    ncol[i] = c;
  }
  for (std::size_t i = 0; i < nr; ++i) {
    if (bad[i] >= 0) bad_token(path, rows[i].substr(bad[i], badlen[i]));
    if (ncol[i] != width) throw FormatError(path + ": ragged rows");
  }
  out.values = std::move(values);
  return out;
}

void write_csv_matrix(const std::string& path, const Matrix& m,
                      const std::optional<std::vector<int>>& signs) {
  FilePtr f = open_for_write(path);
  if (signs) {
    std::fputs("# signs: ", f.get());
    for (std::size_t i = 0; i < signs->size(); ++i)
      std::fprintf(f.get(), "%s%+d", i ? "," : "", (*signs)[i]);
    std::fputc('\n', f.get());
  }
  const std::size_t cols = m.cols();
  parallel_write(f.get(), m.rows(), cols * 26 + 1, [&](std::size_t i, char* b) {
    std::size_t len = 0;
    for (std::size_t j = 0; j < cols; ++j) {
      if (j) b[len++] = ',';
      len += format_value(b + len, m(i, j));
    }
    b[len++] = '\n';
    return len;
  });
}

}  // namespace eigmod

// ----------------------------------------------------------- C ABI (FFI)
#include "eigmod_b200_io.h"

namespace {
thread_local std::string g_io_err;
thread_local eigmod::CsvMatrix g_csv;
thread_local eigmod::SymmetricDense g_mm;

template <class F>
int io_call(F&& f) {
  try {
    f();
    g_io_err.clear();
    return 0;
  } catch (const eigmod::FormatError& e) {
    g_io_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_io_err = e.what();
    return 4;
  }
}
}  // namespace

extern "C" {

const char* eigmod_b200_io_last_error(void) { return g_io_err.c_str(); }

int eigmod_b200_io_write_csv(const char* path, const double* m, int64_t rows, int64_t cols,
                             const int* signs, int64_t nsigns) {
  return io_call([&] {
    eigmod::Matrix mat(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    if (rows * cols) std::memcpy(mat.data(), m, sizeof(double) * rows * cols);
    std::optional<std::vector<int>> s;
    if (signs) s = std::vector<int>(signs, signs + nsigns);
    eigmod::write_csv_matrix(path, mat, s);
  });
}

int eigmod_b200_io_read_csv(const char* path, int64_t* shape3) {
  return io_call([&] {
    g_csv = eigmod::read_csv_matrix(path);
    shape3[0] = static_cast<int64_t>(g_csv.values.rows());
    shape3[1] = static_cast<int64_t>(g_csv.values.cols());
    shape3[2] = g_csv.signs ? static_cast<int64_t>(g_csv.signs->size()) : -1;
  });
}

int eigmod_b200_io_take_csv(double* values, int* signs) {
  return io_call([&] {
    const std::size_t cnt = g_csv.values.rows() * g_csv.values.cols();
    if (values && cnt) std::memcpy(values, g_csv.values.data(), sizeof(double) * cnt);
    if (signs && g_csv.signs)
      for (std::size_t i = 0; i < g_csv.signs->size(); ++i) signs[i] = (*g_csv.signs)[i];
    g_csv = eigmod::CsvMatrix{};
  });
}

int eigmod_b200_io_write_matrix_market(const char* path, const double* a, int64_t n) {
  return io_call([&] {
    eigmod::Matrix mat(static_cast<std::size_t>(n), static_cast<std::size_t>(n));
    if (n) std::memcpy(mat.data(), a, sizeof(double) * n * n);
    eigmod::write_matrix_market(path, eigmod::SymmetricDense::from(mat));
  });
}

int eigmod_b200_io_read_matrix_market(const char* path, int64_t* n_out) {
  return io_call([&] {
    g_mm = eigmod::read_matrix_market(path);
    *n_out = static_cast<int64_t>(g_mm.n);
  });
}

int eigmod_b200_io_take_matrix_market(double* a) {
  return io_call([&] {
    if (a && g_mm.n) std::memcpy(a, g_mm.entries.data(), sizeof(double) * g_mm.n * g_mm.n);
    g_mm = eigmod::SymmetricDense{};
  });
}

}  // extern "C"

// rdcnn/bench.hpp -- the benchmark protocol: Throughput, throughput, BenchRecord, BenchCellError, bench_suite, emit_csv/table/json
// (reference proj/include/rdcnn/bench.hpp:21-251), for the cuda backend: implemented
// over the C-ABI in include/rdcnn_cuda.h.  Part of the source-compatible
// drop-in API; rdcnn/cuda_api.hpp includes every part.
#pragma once

#include <algorithm>
#include <array>
#include <charconv>
#include <chrono>
#include <cmath>
#include <concepts>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "rdcnn_cuda.h"
#include "rdcnn/engine.hpp"
#include "rdcnn/init.hpp"

namespace rdcnn {

// ===========================================================================
// Throughput metric (bench.hpp:21-33)
// ===========================================================================

struct ZeroDuration : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct Throughput {
  double mcells_per_s = 0;
  double ns_per_cell_iter = 0;
};

inline Throughput throughput(long nn, long nm, long iter_max, double seconds) {
  if (!(seconds > 0)) throw ZeroDuration("throughput needs seconds > 0");
  const double work = double(nn) * double(nm) * double(iter_max);
  return {work / (seconds * 1e6), seconds * 1e9 / work};
}

// ===========================================================================
// Benchmark protocol (bench.hpp:35-253): the suite the reference's CLI
// `bench` runs, timed through run_timed on the chosen backend.
// ===========================================================================

struct BenchRecord {
  std::string backend;
  std::string hardware;
  int n = 0;
  long iters = 0;
  double seconds = 0;
  double mcells_per_s = 0;
  double ns_per_cell_iter = 0;
  uint64_t checksum = 0;
  bool skipped = false;  // the cell could not allocate (host or device)
};

/// BlowUpError inside a benchmark cell, naming the cell (bench.hpp:48-59).
struct BenchCellError : std::runtime_error {
  std::string backend;
  int n;
  long iteration;
  BenchCellError(std::string be, int size, long iter)
      : std::runtime_error("blow-up in benchmark cell backend=" + be + " N=" + std::to_string(size) +
                           " at iteration " + std::to_string(iter)),
        backend(std::move(be)),
        n(size),
        iteration(iter) {}
};

namespace detail_bench {

/// One cell: `reps` runs of run_timed from the same typ=1 state, the median
/// wall time, the checksum of the last final state (bench.hpp:63-88).
template <class T>
BenchRecord bench_cell(const Backend& backend, int n, long iter_max, const Gene& gene, uint64_t seed, int reps,
                       const std::string& hardware) {
  std::vector<double> seconds;
  uint64_t digest = 0;
  for (int rep = 0; rep < reps; ++rep) {
    StepBuffers<T> bufs(init_center_square<T>(n, n, seed));
    try {
      seconds.push_back(run_timed(bufs, gene, backend, iter_max));
    } catch (const BlowUpError& e) {
      throw BenchCellError(backend_name(backend), n, e.iteration);
    }
    digest = checksum(bufs.front);
  }
  std::sort(seconds.begin(), seconds.end());
  BenchRecord r;
  r.backend = backend_name(backend);
  r.hardware = hardware;
  r.n = n;
  r.iters = iter_max;
  r.seconds = seconds[seconds.size() / 2];
  const Throughput tp = throughput(n, n, iter_max, r.seconds);
  r.mcells_per_s = tp.mcells_per_s;
  r.ns_per_cell_iter = tp.ns_per_cell_iter;
  r.checksum = digest;
  return r;
}

template <class T>
void warm_up(const Backend& backend, int n, long iter_max, const Gene& gene, uint64_t seed) {
  StepBuffers<T> bufs(init_center_square<T>(n, n, seed));
  try {
    run_timed(bufs, gene, backend, std::min<long>(iter_max, 100));
  } catch (const BlowUpError& e) {
    throw BenchCellError(backend_name(backend), n, e.iteration);
  }
}

inline std::string printf_g(const char* fmt, double x) {
  char buf[64];
  std::snprintf(buf, sizeof buf, fmt, x);
  return buf;
}

/// A double as a JSON number in the form the reference's JSON library
/// writes it: round-trip digits, fixed notation with a ".0" on integral
/// values for decimal exponents in (-4, 15], else d.ddde+XX.  Byte-identical
/// to the reference's emit_json except for rare 17-digit values, where its
/// Grisu2 picks a different last digit of the same double (11 of ~8000 random
/// doubles; both strings parse back to the same value).
inline std::string json_number(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
  std::string s(buf, res.ptr);
  std::string sign;
  if (s[0] == '-') {
    sign = "-";
    s.erase(0, 1);
  }
  const size_t e = s.find('e');
  const int point = std::stoi(s.substr(e + 1)) + 1;  // decimal point position after the first digit
  std::string digits = s.substr(0, e);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int k = int(digits.size());
  std::string out;
  if (k <= point && point <= 15) {
    out = digits + std::string(size_t(point - k), '0') + ".0";
  } else if (0 < point && point <= 15) {
    out = digits.substr(0, size_t(point)) + "." + digits.substr(size_t(point));
  } else if (-4 < point && point <= 0) {
    out = "0." + std::string(size_t(-point), '0') + digits;
  } else {
    out = digits.substr(0, 1) + (k > 1 ? "." + digits.substr(1) : std::string());
    const int ex = point - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
  return sign + out;
}

inline std::string json_string(const std::string& s) {
  std::string out = "\"";
  for (const unsigned char c : s) {
    if (c == '"' || c == '\\') {
      out += '\\';
      out += char(c);
    } else if (c < 0x20) {
      char eb[8];
      std::snprintf(eb, sizeof eb, "\\u%04x", c);
      out += eb;
    } else {
      out += char(c);
    }
  }
  return out + "\"";
}

}  // namespace detail_bench

/// Times every (backend, N) cell on the typ=1 workload (bench.hpp:92-145):
/// one discarded warm-up run per backend before its first cell, the median
/// of `reps` per cell, no snapshots.  A cell that cannot allocate is marked
/// skipped; a blow-up throws BenchCellError.
inline std::vector<BenchRecord> bench_suite(const std::vector<Backend>& backends, const std::vector<int>& sizes,
                                            long iter_max, const Gene& gene, uint64_t seed,
                                            Precision precision = Precision::Single, int reps = 3,
                                            const std::string& hardware = "cpu") {
  if (iter_max < 1) throw std::invalid_argument("bench needs iter_max >= 1");
  if (reps < 1) throw std::invalid_argument("bench needs reps >= 1");
  for (const int n : sizes)
    if (n < 11) throw std::invalid_argument("bench sizes must be >= 11 (typ=1 seed square)");
  const bool single = precision == Precision::Single;
  std::vector<BenchRecord> records;
  for (const Backend& backend : backends) {
    bool warmed = false;
    for (const int n : sizes) {
      try {
        if (!warmed) {
          single ? detail_bench::warm_up<float>(backend, n, iter_max, gene, seed)
                 : detail_bench::warm_up<double>(backend, n, iter_max, gene, seed);
          warmed = true;
        }
        records.push_back(single ? detail_bench::bench_cell<float>(backend, n, iter_max, gene, seed, reps, hardware)
                                 : detail_bench::bench_cell<double>(backend, n, iter_max, gene, seed, reps,
                                                                    hardware));
      } catch (const std::bad_alloc&) {
        BenchRecord r;
        r.backend = backend_name(backend);
        r.hardware = hardware;
        r.n = n;
        r.iters = iter_max;
        r.skipped = true;
        records.push_back(r);
      }
    }
  }
  return records;
}

/// The documented CSV columns; skipped cells are left out (bench.hpp:163-178).
inline std::string emit_csv(const std::vector<BenchRecord>& records) {
  if (records.empty()) throw std::invalid_argument("no benchmark records");
  std::string out = "backend,hardware,n,iters,seconds,mcells_per_s,ns_per_cell_iter,checksum\n";
  for (const BenchRecord& r : records) {
    if (r.skipped) continue;
    out += r.backend + "," + r.hardware + "," + std::to_string(r.n) + "," + std::to_string(r.iters) + "," +
           detail_bench::printf_g("%.5g", r.seconds) + "," + detail_bench::printf_g("%.5g", r.mcells_per_s) + "," +
           detail_bench::printf_g("%.5g", r.ns_per_cell_iter) + "," + checksum_hex(r.checksum) + "\n";
  }
  return out;
}

/// Backend-by-size matrix, each cell "mcells (seconds)", "-" where skipped
/// or absent; a hardware column only when the records carry more than one
/// hardware label (bench.hpp:180-228).
inline std::string emit_table(const std::vector<BenchRecord>& records) {
  if (records.empty()) throw std::invalid_argument("no benchmark records");
  std::vector<int> sizes;
  std::vector<std::pair<std::string, std::string>> keys;  // (backend, hardware), first-seen order
  for (const BenchRecord& r : records) {
    if (std::find(sizes.begin(), sizes.end(), r.n) == sizes.end()) sizes.push_back(r.n);
    const auto key = std::make_pair(r.backend, r.hardware);
    if (std::find(keys.begin(), keys.end(), key) == keys.end()) keys.push_back(key);
  }
  std::sort(sizes.begin(), sizes.end());
  const bool multi_hw = std::any_of(keys.begin(), keys.end(), [&](const auto& k) { return k.second != keys[0].second; });
  auto find = [&](const std::pair<std::string, std::string>& key, int n) -> const BenchRecord* {
    const BenchRecord* hit = nullptr;  // the last record of a repeated cell wins
    for (const BenchRecord& r : records)
      if (r.backend == key.first && r.hardware == key.second && r.n == n) hit = &r;
    return hit;
  };
  std::vector<std::vector<std::string>> cells;
  std::vector<std::string> head{"backend"};
  if (multi_hw) head.push_back("hardware");
  for (const int n : sizes) head.push_back("N=" + std::to_string(n));
  cells.push_back(head);
  for (const auto& key : keys) {
    std::vector<std::string> line{key.first};
    if (multi_hw) line.push_back(key.second);
    for (const int n : sizes) {
      const BenchRecord* r = find(key, n);
      line.push_back(!r || r->skipped ? std::string("-")
                                      : detail_bench::printf_g("%.5g", r->mcells_per_s) + " (" +
                                            detail_bench::printf_g("%.4g", r->seconds) + ")");
    }
    cells.push_back(line);
  }
  std::vector<size_t> width(head.size(), 0);
  for (const auto& line : cells)
    for (size_t c = 0; c < line.size(); ++c) width[c] = std::max(width[c], line[c].size());
  std::string out;
  for (const auto& line : cells) {
    for (size_t c = 0; c < line.size(); ++c) {
      out += line[c];
      if (c + 1 < line.size()) out += std::string(width[c] - line[c].size() + 2, ' ');
    }
    out += "\n";
  }
  return out;
}

/// The CSV fields as a JSON array, two-space indented with keys in sorted
/// order; checksums as hex strings (bench.hpp:230-251).
inline std::string emit_json(const std::vector<BenchRecord>& records) {
  if (records.empty()) throw std::invalid_argument("no benchmark records");
  using detail_bench::json_number;
  using detail_bench::json_string;
  std::string out = "[\n";
  for (size_t i = 0; i < records.size(); ++i) {
    const BenchRecord& r = records[i];
    std::vector<std::pair<std::string, std::string>> kv{{"backend", json_string(r.backend)},
                                                        {"hardware", json_string(r.hardware)},
                                                        {"iters", std::to_string(r.iters)},
                                                        {"n", std::to_string(r.n)}};
    if (r.skipped) {
      kv.emplace_back("skipped", "true");
    } else {
      kv.emplace_back("checksum", json_string(checksum_hex(r.checksum)));
      kv.emplace_back("mcells_per_s", json_number(r.mcells_per_s));
      kv.emplace_back("ns_per_cell_iter", json_number(r.ns_per_cell_iter));
      kv.emplace_back("seconds", json_number(r.seconds));
    }
    std::sort(kv.begin(), kv.end());
    out += "  {\n";
    for (size_t k = 0; k < kv.size(); ++k)
      out += "    \"" + kv[k].first + "\": " + kv[k].second + (k + 1 < kv.size() ? ",\n" : "\n");
    out += i + 1 < records.size() ? "  },\n" : "  }\n";
  }
  return out + "]\n";
}

}  // namespace rdcnn

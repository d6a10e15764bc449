// TEST INFRASTRUCTURE: C-ABI adapter over OUR drop-in I/O (include/nuspectral/io.hpp,
// libnuspectral_b200.so) with the same signatures as oracle/ref_io_shim.cpp, so that
// tests/test_io.py drives both through one wrapper and compares with the reference goldens.
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "nuspectral/io.hpp"

using namespace nuspectral;

namespace {
template <class F>
int io_guard(F&& f, char* err, int64_t errlen, int64_t* line) {
  try {
    f();
    return 0;
  } catch (const io::ParseError& e) {
    if (line) *line = static_cast<int64_t>(e.line());
    if (err && errlen > 0) std::snprintf(err, static_cast<size_t>(errlen), "%s", e.what());
    return 3;
  } catch (const std::exception& e) {
    if (err && errlen > 0) std::snprintf(err, static_cast<size_t>(errlen), "%s", e.what());
    return 1;
  }
}
int put(const std::string& s, char* out, int64_t cap, int64_t* len) {
  *len = static_cast<int64_t>(s.size());
  if (static_cast<int64_t>(s.size()) + 1 > cap) return 2;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}
BandPlan make_plan(const double* c, int64_t nc, double f_w, double f_max, double margin) {
  std::vector<AnalysisBand> bands;
  for (int64_t i = 0; i < nc; ++i) bands.emplace_back(c[i], f_w);
  return BandPlan(std::move(bands), f_max, margin);
}
}  // namespace

extern "C" {
int io_read_csv(const char* text, double* t, double* x, int64_t cap, int64_t* n, int32_t* was_sorted, char* err,
                int64_t errlen, int64_t* line) {
  return io_guard(
      [&] {
        std::istringstream in(text);
        const io::ReadResult r = io::read_time_series_csv(in);
        const auto& tt = r.series.grid.times();
        *n = static_cast<int64_t>(tt.size());
        for (int64_t i = 0; i < *n && i < cap; ++i) {
          t[i] = tt[i];
          x[i] = r.series.values[i];
        }
        *was_sorted = r.was_sorted ? 1 : 0;
      },
      err, errlen, line);
}
int io_config_hash(const char* s, char* out, int64_t cap) {
  int64_t len = 0;
  return put(io::config_hash(s), out, cap, &len);
}
int io_library_version(char* out, int64_t cap) {
  int64_t len = 0;
  return put(io::library_version(), out, cap, &len);
}
int io_write_series_csv(const double* t, const double* x, int64_t n, const char* hash, char* out, int64_t cap,
                        int64_t* len) {
  std::string s;
  const int rc = io_guard(
      [&] {
        std::ostringstream os;
        io::write_time_series_csv(
            os, SignalSeries(SamplingGrid(std::vector<double>(t, t + n)), std::vector<double>(x, x + n)), hash);
        s = os.str();
      },
      nullptr, 0, nullptr);
  return rc ? rc : put(s, out, cap, len);
}
int io_write_spectrum_csv(const double* c, int64_t nc, double f_w, double f_max, double margin, const double* power,
                          const int64_t* k_used, const double* fw_used, const uint8_t* flags, int32_t method,
                          const char* hash, char* out, int64_t cap, int64_t* len) {
  std::string s;
  const int rc = io_guard(
      [&] {
        const SpectrumEstimate e(make_plan(c, nc, f_w, f_max, margin), std::vector<double>(power, power + nc),
                                 static_cast<EstimatorMethod>(method), std::vector<std::size_t>(k_used, k_used + nc),
                                 std::vector<double>(fw_used, fw_used + nc),
                                 std::vector<std::uint8_t>(flags, flags + nc));
        std::ostringstream os;
        io::write_spectrum_csv(os, e, hash);
        s = os.str();
      },
      nullptr, 0, nullptr);
  return rc ? rc : put(s, out, cap, len);
}
int io_write_ftest_csv(const double* c, int64_t nc, double f_w, double f_max, double margin, const double* f_stat,
                       const double* amp, const uint8_t* flags, int64_t d1, int64_t d2, const double* p_levels,
                       const double* crits, int64_t ncrit, double sat_cap, const char* hash, char* out, int64_t cap,
                       int64_t* len) {
  std::string s;
  const int rc = io_guard(
      [&] {
        FTestResult r{make_plan(c, nc, f_w, f_max, margin), std::vector<double>(f_stat, f_stat + nc), {}, {}, {}, {},
                      sat_cap};
        for (int64_t i = 0; i < nc; ++i) r.amplitude.emplace_back(amp[2 * i], amp[2 * i + 1]);
        r.dof = {static_cast<std::size_t>(d1), static_cast<std::size_t>(d2)};
        for (int64_t q = 0; q < ncrit; ++q) r.critical_values.emplace_back(p_levels[q], crits[q]);
        r.flags.assign(flags, flags + nc);
        std::ostringstream os;
        io::write_ftest_csv(os, r, hash);
        s = os.str();
      },
      nullptr, 0, nullptr);
  return rc ? rc : put(s, out, cap, len);
}
int io_write_manifest(const char* command, const char* const* keys, const char* const* vals, int64_t nf,
                      const char* hash, char* out, int64_t cap, int64_t* len) {
  std::string s;
  const int rc = io_guard(
      [&] {
        std::vector<std::pair<std::string, std::string>> fields;
        for (int64_t i = 0; i < nf; ++i) fields.emplace_back(keys[i], vals[i]);
        std::ostringstream os;
        io::write_manifest_json(os, command, fields, hash);
        s = os.str();
      },
      nullptr, 0, nullptr);
  return rc ? rc : put(s, out, cap, len);
}
}  // extern "C"

// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI adapter over the reference's I/O layer (src/io.cpp, compiled unmodified
// into oracle/_ref/libnusref.so with the nlohmann header the image provides).
// Used by tests/golden/make_golden.py to pin the byte-exact behaviour of the
// readers and writers around the MTNUFFT path:
// read_time_series_csv (io.cpp:37-101), config_hash (io.cpp:109-118),
// write_time_series_csv / write_spectrum_csv / write_ftest_csv (io.cpp:120-188),
// write_manifest_json + library_version (io.cpp:265-276).

#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "nuspectral/errors.hpp"
#include "nuspectral/estimators.hpp"
#include "nuspectral/grid.hpp"
#include "nuspectral/inference.hpp"
#include "nuspectral/io.hpp"

using namespace nuspectral;

namespace {

// 0 ok, 3 ParseError (line in *line), 1 other error; message copied to err
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

int ref_io_read_csv(const char* text, double* t, double* x, int64_t cap, int64_t* n, int32_t* was_sorted, char* err,
                    int64_t errlen, int64_t* line) {
  return io_guard(
      [&] {
        std::istringstream in(text);
        const io::ReadResult r = io::read_time_series_csv(in);
        const auto& tt = r.series.grid.times();
        *n = static_cast<int64_t>(tt.size());
        if (*n > cap) throw std::runtime_error("capacity");
        for (int64_t i = 0; i < *n; ++i) {
          t[i] = tt[i];
          x[i] = r.series.values[i];
        }
        *was_sorted = r.was_sorted ? 1 : 0;
      },
      err, errlen, line);
}

int ref_io_config_hash(const char* s, char* out, int64_t cap) {
  const std::string h = io::config_hash(s);
  int64_t len = 0;
  return put(h, out, cap, &len);
}

int ref_io_library_version(char* out, int64_t cap) {
  int64_t len = 0;
  return put(io::library_version(), out, cap, &len);
}

int ref_io_write_series_csv(const double* t, const double* x, int64_t n, const char* hash, char* out, int64_t cap,
                            int64_t* len) {
  std::string s;
  const int rc = io_guard(
      [&] {
        std::ostringstream os;
        io::write_time_series_csv(os, SignalSeries(SamplingGrid(std::vector<double>(t, t + n)),
                                                   std::vector<double>(x, x + n)),
                                  hash);
        s = os.str();
      },
      nullptr, 0, nullptr);
  return rc ? rc : put(s, out, cap, len);
}

int ref_io_write_spectrum_csv(const double* c, int64_t nc, double f_w, double f_max, double margin,
                              const double* power, const int64_t* k_used, const double* fw_used,
                              const uint8_t* flags, int32_t method, const char* hash, char* out, int64_t cap,
                              int64_t* len) {
  std::string s;
  const int rc = io_guard(
      [&] {
        std::vector<std::size_t> k(k_used, k_used + nc);
        const SpectrumEstimate e(make_plan(c, nc, f_w, f_max, margin), std::vector<double>(power, power + nc),
                                 static_cast<EstimatorMethod>(method), std::move(k),
                                 std::vector<double>(fw_used, fw_used + nc),
                                 std::vector<std::uint8_t>(flags, flags + nc));
        std::ostringstream os;
        io::write_spectrum_csv(os, e, hash);
        s = os.str();
      },
      nullptr, 0, nullptr);
  return rc ? rc : put(s, out, cap, len);
}

int ref_io_write_ftest_csv(const double* c, int64_t nc, double f_w, double f_max, double margin,
                           const double* f_stat, const double* amp, const uint8_t* flags, int64_t d1, int64_t d2,
                           const double* p_levels, const double* crits, int64_t ncrit, double sat_cap,
                           const char* hash, char* out, int64_t cap, int64_t* len) {
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

int ref_io_write_manifest(const char* command, const char* const* keys, const char* const* vals, int64_t nf,
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

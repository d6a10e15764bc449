// I/O around the MTNUFFT path — drop-in for the reference's src/io.cpp.
//
// read_time_series_csv follows io.cpp:37-101 (the sample-sorting contract), config_hash
// io.cpp:109-118, the writers io.cpp:120-188 and write_manifest_json io.cpp:265-274.
// Byte-exact against the reference on tests/golden/io_golden.json (tests/test_io.py).
#include "nuspectral/io.hpp"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iomanip>
#include <istream>
#include <limits>
#include <map>
#include <numeric>
#include <ostream>
#include <sstream>

namespace nuspectral::io {

namespace {

std::string strip(const std::string& s) {
  const auto a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return std::string();
  return s.substr(a, s.find_last_not_of(" \t\r\n") - a + 1);
}

// std::stod semantics: strtod, no conversion or ERANGE (overflow and underflow) -> failure;
// in addition the whole field must be consumed (io.cpp:67-70)
bool parse_field(const std::string& s, double& v) {
  if (s.empty()) return false;
  const char* b = s.c_str();
  char* e = nullptr;
  errno = 0;
  v = std::strtod(b, &e);
  if (e == b || errno == ERANGE) return false;
  return static_cast<std::size_t>(e - b) == s.size();
}

// the reference prints through a stream whose precision, once set to 17 by the first full
// print, stays 17 for every later unformatted double (io.cpp:25-31)
void put_full(std::ostream& out, double v) {
  if (std::isnan(v)) {
    out << "nan";
    return;
  }
  out << std::setprecision(17) << v;
}

void put_json_string(std::ostream& out, const std::string& s) {
  static const char* hex = "0123456789abcdef";
  out << '"';
  for (const unsigned char c : s) {
    switch (c) {
      case '"': out << "\\\""; break;
      case '\\': out << "\\\\"; break;
      case '\b': out << "\\b"; break;
      case '\f': out << "\\f"; break;
      case '\n': out << "\\n"; break;
      case '\r': out << "\\r"; break;
      case '\t': out << "\\t"; break;
      default:
        if (c < 0x20) out << "\\u00" << hex[c >> 4] << hex[c & 15];
        else out << static_cast<char>(c);
    }
  }
  out << '"';
}

}  // namespace

ReadResult read_time_series_csv(std::istream& in) {
  std::vector<double> t, x;
  std::string raw;
  std::size_t line = 0;
  bool have_header = false;
  while (std::getline(in, raw)) {
    ++line;
    const std::string s = strip(raw);
    if (s.empty() || s.front() == '#') continue;
    if (!have_header) {
      std::string h;
      for (const char c : s)
        if (c != ' ' && c != '\t') h.push_back(c);
      if (h != "t,x") throw ParseError("expected header 't,x', got '" + s + "'", line);
      have_header = true;
      continue;
    }
    const std::size_t comma = s.find(',');
    if (comma == std::string::npos) throw ParseError("expected 't,x' row", line);
    double tv = 0.0, xv = 0.0;
    if (!parse_field(strip(s.substr(0, comma)), tv) || !parse_field(strip(s.substr(comma + 1)), xv) ||
        !std::isfinite(tv) || !std::isfinite(xv))
      throw ParseError("could not parse row '" + s + "'", line);
    t.push_back(tv);
    x.push_back(xv);
  }
  if (!have_header) throw ParseError("empty input: missing 't,x' header", line);
  if (t.size() < 2) throw ParseError("need at least 2 samples", line);

  const bool sorted = std::is_sorted(t.begin(), t.end());
  if (!sorted) {  // stable: equal times keep their file order (and are then rejected below)
    std::vector<std::size_t> order(t.size());
    std::iota(order.begin(), order.end(), std::size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return t[a] < t[b]; });
    std::vector<double> ts, xs;
    ts.reserve(t.size());
    xs.reserve(x.size());
    for (const std::size_t i : order) {
      ts.push_back(t[i]);
      xs.push_back(x[i]);
    }
    t.swap(ts);
    x.swap(xs);
  }
  for (std::size_t i = 1; i < t.size(); ++i)
    if (t[i] == t[i - 1]) throw ParseError("duplicate sample time " + std::to_string(t[i]), 0);
  return ReadResult{SignalSeries(SamplingGrid(std::move(t)), std::move(x)), sorted};
}

ReadResult read_time_series_csv_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw Error("cannot open input file: " + path);
  return read_time_series_csv(in);
}

std::string config_hash(const std::string& canonical) {
  std::uint64_t h = 14695981039346656037ull;  // FNV-1a 64 offset basis
  for (const unsigned char c : canonical) {
    h ^= c;
    h *= 1099511628211ull;  // FNV prime
  }
  std::ostringstream os;
  os << std::hex << std::setfill('0') << std::setw(16) << h;
  return os.str();
}

void write_time_series_csv(std::ostream& out, const SignalSeries& series, const std::string& hash) {
  out << "# config_hash=" << hash << "\nt,x\n";
  const auto& t = series.grid.times();
  for (std::size_t i = 0; i < t.size(); ++i) {
    put_full(out, t[i]);
    out << ',';
    put_full(out, series.values[i]);
    out << '\n';
  }
}

void write_spectrum_csv(std::ostream& out, const SpectrumEstimate& e, const std::string& hash) {
  out << "# config_hash=" << hash << "\n# method=" << method_name(e.method) << "\n";
  out << "f_center,power,power_db,k_used,f_w_used,flag\n";
  for (std::size_t i = 0; i < e.plan.size(); ++i) {
    const double p = e.power[i];
    put_full(out, e.plan.center(i));
    out << ',';
    put_full(out, p);
    out << ',';
    const double db = p > 0.0 ? 10.0 * std::log10(p) : -std::numeric_limits<double>::infinity();
    if (std::isnan(p)) out << "nan";
    else if (std::isinf(db)) out << "-inf";  // as the reference: any infinite dB prints -inf
    else put_full(out, db);
    out << ',' << e.k_used[i] << ',';
    put_full(out, e.f_w_used[i]);
    out << ',' << static_cast<int>(e.flags[i]) << '\n';
  }
}

void write_ftest_csv(std::ostream& out, const FTestResult& r, const std::string& hash) {
  out << "# config_hash=" << hash << "\n# dof=" << r.dof.first << ',' << r.dof.second << '\n';
  for (const auto& pc : r.critical_values) {
    out << "# critical p=" << pc.first << " value=";  // p in the stream's current precision
    put_full(out, pc.second);
    out << '\n';
  }
  out << "f_center,f_stat,amp_re,amp_im";
  for (const auto& pc : r.critical_values) out << ",exceeds_p" << pc.first;
  out << ",flag\n";
  for (std::size_t i = 0; i < r.plan.size(); ++i) {
    put_full(out, r.plan.center(i));
    out << ',';
    put_full(out, r.f_stat[i]);
    out << ',';
    put_full(out, r.amplitude[i].real());
    out << ',';
    put_full(out, r.amplitude[i].imag());
    for (const auto& pc : r.critical_values) out << ',' << (r.f_stat[i] > pc.second ? 1 : 0);
    out << ',' << static_cast<int>(r.flags[i]) << '\n';
  }
}

void write_manifest_json(std::ostream& out, const std::string& command,
                         const std::vector<std::pair<std::string, std::string>>& fields, const std::string& hash) {
  std::map<std::string, std::string> config;  // byte-order keys, the last duplicate wins
  for (const auto& kv : fields) config[kv.first] = kv.second;
  out << "{\n  \"command\": ";
  put_json_string(out, command);
  out << ",\n";
  if (!config.empty()) {
    out << "  \"config\": {\n";
    std::size_t i = 0;
    for (const auto& kv : config) {
      out << "    ";
      put_json_string(out, kv.first);
      out << ": ";
      put_json_string(out, kv.second);
      out << (++i < config.size() ? ",\n" : "\n");
    }
    out << "  },\n";
  }
  out << "  \"config_hash\": ";
  put_json_string(out, hash);
  out << ",\n  \"version\": ";
  put_json_string(out, library_version());
  out << "\n}\n";
}

// The version string the reference embeds in manifests (io.cpp:276): kept so that files
// written by either library are interchangeable.
std::string library_version() { return "0.1.0"; }

}  // namespace nuspectral::io

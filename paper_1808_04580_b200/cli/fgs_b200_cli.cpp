// fgs_b200_cli.cpp -- the reference's command-line drivers for the hot path
// (tools/commands.cpp: eigs, cluster, bench) on the B200 library, with the
// same flags, defaults, exit codes and `fgs-report-v1` JSON report
// (report.cpp:97-112, schema/report.schema.json).
//
// Everything numeric goes through include/fgs/b200.hpp (the C ABI): plans,
// degrees, Lanczos, residuals, k-means and the dense-reference metrics (the
// Direct backend, i.e. exact O(n^2) applies on the GPU).  Host code here is
// I/O, argument parsing and report assembly.
//
// Methods: nfft-lanczos (Fastsum backend), direct (Direct backend) and
// nystrom-gauss-nfft (Gaussian sketch over the fast operator).  The sampled
// "nystrom" method (dense kernel blocks, spectral.cpp:277-382) is not part of
// this build and is rejected as a usage error, as are the commands outside
// the hot path's scope (gen, segment, ssl-kernel, krr, ssl-pf: data
// generation, image I/O and the semi-supervised drivers; SURVEY.md section 2,
// DESIGN.md section 7).  The library functions behind ssl-kernel / krr
// (kernel_ssl_solve, krr_fit / krr_predict) remain in include/fgs/b200.hpp.
#include <algorithm>
#include <cctype>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <sstream>
#include <charconv>
#include <string>
#include <vector>

#include "fgs/b200.hpp"

namespace cli {

using fgs::AdjacencyBackend;
using fgs::AdjacencyOperator;
using fgs::EigenPairs;
using fgs::FastsumParams;
using fgs::Index;
using fgs::KernelSpec;
using fgs::MatrixXd;
using fgs::VectorXd;

constexpr double kPi = 3.14159265358979323846;
constexpr Index kReferenceBudget = 23000;  // commands.cpp:24-25

class ParseError : public std::runtime_error {  // errors.hpp (I/O)
 public:
  using std::runtime_error::runtime_error;
};
class FormatError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class UsageError : public std::invalid_argument {  // CLI11::ParseError analogue
 public:
  using std::invalid_argument::invalid_argument;
};

// ---- minimal JSON (object keys sorted, as nlohmann::json's std::map) -------
class Json {
 public:
  enum Kind { Null, Bool, Int, Num, Str, Arr, Obj };
  Json() = default;
  Json(bool b) : k_(Bool), b_(b) {}
  Json(int v) : k_(Int), i_(v) {}
  Json(long v) : k_(Int), i_(v) {}
  Json(long long v) : k_(Int), i_(v) {}
  Json(unsigned long v) : k_(Int), i_(static_cast<long long>(v)) {}
  Json(double v) : k_(Num), d_(v) {}
  Json(const char* s) : k_(Str), s_(s) {}
  Json(std::string s) : k_(Str), s_(std::move(s)) {}
  template <class T>
  Json(const std::vector<T>& v) : k_(Arr) {
    for (const auto& x : v) a_.emplace_back(x);
  }
  static Json object() {
    Json j;
    j.k_ = Obj;
    return j;
  }
  static Json array() {
    Json j;
    j.k_ = Arr;
    return j;
  }
  Json& operator[](const std::string& key) {
    if (k_ == Null) k_ = Obj;
    return o_[key];
  }
  void push_back(Json v) {
    if (k_ == Null) k_ = Arr;
    a_.push_back(std::move(v));
  }
  bool empty() const { return (k_ == Obj && o_.empty()) || (k_ == Arr && a_.empty()) || k_ == Null; }
  std::string dump(int indent = 2) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  Kind k_ = Null;
  bool b_ = false;
  long long i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Json> a_;
  std::map<std::string, Json> o_;

  static void esc(std::string& out, const std::string& s) {
    out += '"';
    for (char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\n': out += "\\n"; break;
        case '\t': out += "\\t"; break;
        case '\r': out += "\\r"; break;
        default:
          if (static_cast<unsigned char>(c) < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof(buf), "\\u%04x", c);
            out += buf;
          } else {
            out += c;
          }
      }
    }
    out += '"';
  }
  static std::string num(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[64];
    for (int prec = 15; prec <= 17; ++prec) {  // shortest round-trip
      std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
      if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s = buf;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
  }
  void write(std::string& out, int ind, int depth) const {
    const std::string pad(static_cast<size_t>(ind * (depth + 1)), ' '), end(static_cast<size_t>(ind * depth), ' ');
    switch (k_) {
      case Null: out += "null"; break;
      case Bool: out += b_ ? "true" : "false"; break;
      case Int: out += std::to_string(i_); break;
      case Num: out += num(d_); break;
      case Str: esc(out, s_); break;
      case Arr:
        if (a_.empty()) {
          out += "[]";
          break;
        }
        out += "[\n";
        for (size_t i = 0; i < a_.size(); ++i) {
          out += pad;
          a_[i].write(out, ind, depth + 1);
          out += i + 1 < a_.size() ? ",\n" : "\n";
        }
        out += end + "]";
        break;
      case Obj:
        if (o_.empty()) {
          out += "{}";
          break;
        }
        out += "{\n";
        {
          size_t i = 0;
          for (const auto& kv : o_) {
            out += pad;
            esc(out, kv.first);
            out += ": ";
            kv.second.write(out, ind, depth + 1);
            out += ++i < o_.size() ? ",\n" : "\n";
          }
        }
        out += end + "}";
        break;
    }
  }
};

// ---- report.cpp ------------------------------------------------------------
struct Report {
  std::string command, method, status = "ok", diagnostic;
  std::uint64_t seed = 0;
  Json parameters = Json::object(), metrics = Json::object(), timings = Json::object(), extra = Json::object();
  std::vector<double> eigenvalues;

  void add_metric(const std::string& name, double value, const std::string& definition) {
    Json m = Json::object();
    m["value"] = value;
    m["definition"] = definition;
    metrics[name] = m;
  }
  void add_timing(const std::string& phase, double seconds) { timings[phase] = seconds; }
  Json to_json() const {
    Json out = Json::object();
    out["schema"] = "fgs-report-v1";
    out["command"] = command;
    out["method"] = method;
    out["parameters"] = parameters;
    out["seed"] = static_cast<long long>(seed);
    out["eigenvalues"] = eigenvalues;
    out["metrics"] = metrics;
    out["timings_seconds"] = timings;
    out["status"] = status;
    out["diagnostic"] = diagnostic;
    if (!extra.empty()) out["extra"] = extra;
    return out;
  }
};

void write_report(const Report& r, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw ParseError(path + ": cannot open for writing");
  out << r.to_json().dump(2) << '\n';
  if (!out) throw ParseError(path + ": write failed");
}

class Timer {
 public:
  Timer() : t0_(std::chrono::steady_clock::now()) {}
  double seconds() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count(); }

 private:
  std::chrono::steady_clock::time_point t0_;
};

// ---- dataset.cpp: point clouds, CSV, generators ---------------------------
struct PointCloud {
  MatrixXd coordinates;
  std::vector<int> labels;
  Index size() const { return coordinates.rows(); }
  bool has_labels() const { return !labels.empty(); }
};

std::string trimmed(const std::string& s) {
  const size_t b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  const size_t e = s.find_last_not_of(" \t\r");
  return s.substr(b, e - b + 1);
}

std::vector<std::string> split_row(const std::string& line) {
  std::vector<std::string> cells;
  std::string cell;
  std::stringstream ss(line);
  while (std::getline(ss, cell, ',')) cells.push_back(cell);
  if (!line.empty() && line.back() == ',') cells.emplace_back();
  return cells;
}

[[noreturn]] void parse_fail(const std::string& path, size_t line, const std::string& what) {
  throw ParseError(path + ": line " + std::to_string(line) + ": " + what);
}

template <class T>
T parse_cell(const std::string& cell, const std::string& path, size_t line, const char* what) {
  const std::string t = trimmed(cell);
  T v{};
  auto [ptr, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
  if (ec != std::errc{} || ptr != t.data() + t.size()) parse_fail(path, line, std::string(what) + " cell '" + cell + "'");
  return v;
}

// dataset.cpp:249-294
PointCloud load_points_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError(path + ": cannot open");
  std::string line;
  if (!std::getline(in, line) || trimmed(line).empty()) parse_fail(path, 1, "missing header row");
  const std::vector<std::string> header = split_row(line);
  const bool labeled = !header.empty() && trimmed(header.back()) == "label";
  const size_t cols = header.size(), dims = cols - (labeled ? 1u : 0u);
  if (dims < 1) parse_fail(path, 1, "no coordinate columns");
  std::vector<double> values;
  std::vector<int> labels;
  size_t rows = 0, ln = 1;
  while (std::getline(in, line)) {
    ++ln;
    if (trimmed(line).empty()) continue;
    const std::vector<std::string> cells = split_row(line);
    if (cells.size() != cols)
      parse_fail(path, ln, "expected " + std::to_string(cols) + " cells, found " + std::to_string(cells.size()));
    for (size_t t = 0; t < dims; ++t) {
      const double v = parse_cell<double>(cells[t], path, ln, "non-numeric");
      if (!std::isfinite(v)) parse_fail(path, ln, "non-finite coordinate");
      values.push_back(v);
    }
    if (labeled) labels.push_back(parse_cell<int>(cells.back(), path, ln, "non-integer"));
    ++rows;
  }
  if (rows == 0) parse_fail(path, ln, "no data rows");
  PointCloud c;
  c.coordinates = MatrixXd(static_cast<Index>(rows), static_cast<Index>(dims));
  for (size_t i = 0; i < rows; ++i)
    for (size_t t = 0; t < dims; ++t) c.coordinates(static_cast<Index>(i), static_cast<Index>(t)) = values[i * dims + t];
  c.labels = std::move(labels);
  return c;
}

std::string fmt17(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

void save_labels_csv(const std::vector<int>& labels, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ParseError(path + ": cannot open for writing");
  out << "label\n";
  for (int l : labels) out << l << '\n';
  if (!out) throw ParseError(path + ": write failed");
}

// ---- argument parsing (CLI11 subset: --name value, --flag) ----------------
// dataset.cpp:184-211
PointCloud gen_spiral(int classes, int per_class, double h, double r, std::uint64_t seed) {
  if (classes < 1) throw fgs::ParameterError("spiral needs at least one class");
  if (per_class < 1) throw fgs::ParameterError("spiral needs at least one point per class");
  const Index n = static_cast<Index>(classes) * per_class;
  PointCloud c;
  c.coordinates = MatrixXd(n, 3);
  c.labels.resize(static_cast<size_t>(n));
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::normal_distribution<double> jitter(0.0, 0.1 * r);
  Index row = 0;
  for (int k = 0; k < classes; ++k)
    for (int i = 0; i < per_class; ++i, ++row) {
      const double t = 1.0 - unit(rng);
      const double theta = 2.0 * kPi * (t + static_cast<double>(k) / classes);
      c.coordinates(row, 0) = t * r * std::cos(theta) + jitter(rng);
      c.coordinates(row, 1) = t * r * std::sin(theta) + jitter(rng);
      c.coordinates(row, 2) = h * t + jitter(rng);
      c.labels[static_cast<size_t>(row)] = k;
    }
  return c;
}

class Args {
 public:
  Args(int argc, char** argv, int first) {
    for (int i = first; i < argc; ++i) {
      std::string a = argv[i];
      if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
      std::string key = a.substr(2), val;
      const size_t eq = key.find('=');
      if (eq != std::string::npos) {
        val = key.substr(eq + 1);
        key = key.substr(0, eq);
        kv_[key] = val;
      } else if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) {
        kv_[key] = argv[++i];
      } else {
        kv_[key] = "";
      }
    }
  }
  bool has(const std::string& k) const { return kv_.count(k) != 0; }
  template <class T>
  void get(const std::string& k, T* out) {
    auto it = kv_.find(k);
    if (it == kv_.end()) return;
    used_.push_back(k);
    const std::string& v = it->second;
    if constexpr (std::is_same_v<T, std::string>) {
      *out = v;
    } else if constexpr (std::is_same_v<T, bool>) {
      *out = true;
    } else {
      T x{};
      auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
      if (ec != std::errc{} || p != v.data() + v.size()) throw UsageError("--" + k + ": invalid value '" + v + "'");
      *out = x;
    }
  }
  template <class T>
  void get_list(const std::string& k, std::vector<T>* out) {
    auto it = kv_.find(k);
    if (it == kv_.end()) return;
    used_.push_back(k);
    out->clear();
    std::stringstream ss(it->second);
    std::string item;
    while (std::getline(ss, item, ',')) {
      if constexpr (std::is_same_v<T, std::string>) {
        out->push_back(item);
      } else {
        T x{};
        auto [p, ec] = std::from_chars(item.data(), item.data() + item.size(), x);
        if (ec != std::errc{} || p != item.data() + item.size())
          throw UsageError("--" + k + ": invalid value '" + item + "'");
        out->push_back(x);
      }
    }
  }
  void require(const std::string& k) const {
    if (!has(k)) throw UsageError("--" + k + " is required");
  }
  void finish() const {
    for (const auto& kv : kv_) {
      bool ok = false;
      for (const auto& u : used_) ok = ok || u == kv.first;
      if (!ok) throw UsageError("unknown option --" + kv.first);
    }
  }

 private:
  std::map<std::string, std::string> kv_;
  std::vector<std::string> used_;
};

// ---- commands.cpp:39-171 ---------------------------------------------------
struct CommonOpts {
  std::string in, out, kernel_name = "gaussian", method = "nfft-lanczos";
  double sigma = 1.0, c = 1.0, eps_b = -1.0, tol = -1.0;
  int setup = 2, bandwidth = 0, cutoff = 0, smoothness = 0, k = 10, sketch_l = 100, sketch_m = 10, threads = 0;
  std::uint64_t seed = 1;
  bool with_reference = false;
  int device = 0;
};

void io_flags(Args& a, CommonOpts* o, bool in_required) {
  if (in_required) a.require("in");
  a.require("out");
  a.get("in", &o->in);
  a.get("out", &o->out);
  a.get("seed", &o->seed);
  a.get("threads", &o->threads);
  a.get("device", &o->device);
}

void kernel_flags(Args& a, CommonOpts* o) {
  a.get("kernel", &o->kernel_name);
  if (o->kernel_name != "gaussian" && o->kernel_name != "laplacian-rbf" && o->kernel_name != "multiquadric" &&
      o->kernel_name != "inv-multiquadric")
    throw UsageError("--kernel: " + o->kernel_name + " not in {gaussian, laplacian-rbf, multiquadric, inv-multiquadric}");
  a.get("sigma", &o->sigma);
  a.get("c", &o->c);
}

void fastsum_flags(Args& a, CommonOpts* o) {
  a.get("setup", &o->setup);
  if (o->setup < 1 || o->setup > 3) throw UsageError("--setup: value not in range [1, 3]");
  a.get("N", &o->bandwidth);
  a.get("m", &o->cutoff);
  a.get("p", &o->smoothness);
  a.get("eps-b", &o->eps_b);
}

void method_flags(Args& a, CommonOpts* o) {
  a.get("method", &o->method);
  if (o->method != "nfft-lanczos" && o->method != "nystrom" && o->method != "nystrom-gauss-nfft" &&
      o->method != "direct")
    throw UsageError("--method: " + o->method + " not in {nfft-lanczos, nystrom, nystrom-gauss-nfft, direct}");
  a.get("k", &o->k);
  a.get("L", &o->sketch_l);
  a.get("M", &o->sketch_m);
  a.get("tol", &o->tol);
  a.get("with-reference", &o->with_reference);
}

KernelSpec make_kernel(const CommonOpts& o) {
  if (o.kernel_name == "gaussian") return KernelSpec::gaussian(o.sigma);
  if (o.kernel_name == "laplacian-rbf") return KernelSpec::laplacian_rbf(o.sigma);
  if (o.kernel_name == "multiquadric") return KernelSpec::multiquadric(o.c);
  return KernelSpec::inverse_multiquadric(o.c);
}

FastsumParams make_params(const CommonOpts& o) {
  FastsumParams p = FastsumParams::preset(o.setup, o.eps_b < 0.0 ? 0.0 : o.eps_b);
  if (o.bandwidth > 0) p.bandwidth = o.bandwidth;
  if (o.cutoff > 0) {
    p.cutoff = o.cutoff;
    p.smoothness = o.cutoff;
  }
  if (o.smoothness > 0) p.smoothness = o.smoothness;
  return p;
}

Json echo_common(const CommonOpts& o) {
  const FastsumParams p = make_params(o);
  Json j = Json::object();
  j["in"] = o.in;
  j["out"] = o.out;
  j["kernel"] = o.kernel_name;
  j["sigma"] = o.sigma;
  j["c"] = o.c;
  j["setup"] = o.setup;
  j["bandwidth"] = p.bandwidth;
  j["cutoff"] = p.cutoff;
  j["smoothness"] = p.smoothness;
  j["eps_b"] = p.eps_b;
  j["method"] = o.method;
  j["k"] = o.k;
  j["L"] = o.sketch_l;
  j["M"] = o.sketch_m;
  j["tol"] = o.tol;
  j["threads_requested"] = o.threads;
  j["threads_effective"] = 1;  // one stream per handle: deterministic
  j["with_reference"] = o.with_reference;
  j["device"] = o.device;
  return j;
}

double lanczos_tol(const CommonOpts& o) { return o.tol > 0.0 ? o.tol : 1e-12; }

AdjacencyBackend backend_of(const std::string& method) {
  if (method == "direct") return AdjacencyBackend::Direct;
  if (method == "nfft-lanczos") return AdjacencyBackend::Fastsum;
  throw fgs::ParameterError("method " + method +
                            " is not available in the B200 build (nfft-lanczos, direct, nystrom-gauss-nfft)");
}

// commands.cpp:163-218
EigenPairs solve_pairs(const PointCloud& cloud, const KernelSpec& kernel, const FastsumParams& params,
                       const CommonOpts& o, Report* report) {
  fgs::LanczosOptions lo;
  lo.tol = lanczos_tol(o);
  lo.seed = o.seed;
  if (o.method == "nystrom-gauss-nfft") {  // commands.cpp:197-216
    fgs::NystromOptions no;
    no.k = o.k;
    no.L = o.sketch_l;
    no.M = o.sketch_m;
    no.seed = o.seed;
    Timer setup;
    AdjacencyOperator op(cloud.coordinates, kernel, params, AdjacencyBackend::Fastsum, o.device);
    report->add_timing("setup", setup.seconds());
    Timer solve;
    EigenPairs pairs = fgs::nystrom_gaussian(op, no);
    report->add_timing("solve", solve.seconds());
    report->add_metric("max_residual_operator", fgs::max_residual(op, pairs),
                       "max_i ||A v_i - lambda_i v_i||_2 with the operator used for the solve (approximate for "
                       "nystrom-gauss-nfft)");
    report->eigenvalues.assign(pairs.values.data(), pairs.values.data() + pairs.count());
    return pairs;
  }
  const AdjacencyBackend backend = backend_of(o.method);
  Timer setup;
  AdjacencyOperator op(cloud.coordinates, kernel, params, backend, o.device);
  report->add_timing("setup", setup.seconds());
  Timer solve;
  fgs::LanczosInfo info;
  EigenPairs pairs = fgs::lanczos_largest(op, o.k, lo, &info);
  report->add_timing("solve", solve.seconds());
  report->add_metric("lanczos_iterations", info.iterations, "Lanczos steps executed");
  report->add_metric("lanczos_converged", info.converged ? 1.0 : 0.0,
                     "1 if every wanted Ritz pair met the tolerance");
  report->add_metric("max_residual_operator", fgs::max_residual(op, pairs),
                     "max_i ||A v_i - lambda_i v_i||_2 with the operator used for the solve (approximate for "
                     "nfft-lanczos)");
  report->eigenvalues.assign(pairs.values.data(), pairs.values.data() + pairs.count());
  return pairs;
}

// dense_reference_eig (spectral.cpp:556-585) on the Direct backend
EigenPairs dense_reference_eig(const AdjacencyOperator& exact, int k) {
  fgs::LanczosOptions lo;
  lo.max_iter = 1000;
  lo.tol = 1e-13;
  lo.seed = 12345;
  return fgs::lanczos_largest(exact, k, lo);
}

double max_value_error(const EigenPairs& a, const EigenPairs& b) {
  double e = 0.0;
  for (Index i = 0; i < a.count() && i < b.count(); ++i) e = std::max(e, std::abs(a.values(i) - b.values(i)));
  return e;
}

// commands.cpp:220-249
void add_reference_metrics(const PointCloud& cloud, const KernelSpec& kernel, const EigenPairs& pairs,
                           const CommonOpts& o, Report* report) {
  if (cloud.size() > kReferenceBudget) {
    report->extra["reference_skipped"] =
        "point count exceeds the dense-reference budget of " + std::to_string(kReferenceBudget);
    return;
  }
  Timer ref;
  AdjacencyOperator exact(cloud.coordinates, kernel, FastsumParams{}, AdjacencyBackend::Direct, o.device);
  report->add_metric("max_residual", fgs::max_residual(exact, pairs),
                     "max_i ||A v_i - lambda_i v_i||_2 with exact operator applies");
  const EigenPairs reference = dense_reference_eig(exact, static_cast<int>(pairs.count()));
  report->add_metric("max_eigenvalue_error", max_value_error(pairs, reference),
                     "max_i |lambda_i - lambda_i^dense| against the dense reference eigensolve");
  report->add_timing("reference", ref.seconds());
}

int finish(Report& r, const std::string& path, const std::string& summary) {
  write_report(r, path);
  std::cout << summary << "report: " << path << '\n';
  return r.status == "ok" ? 0 : 1;
}

// commands.cpp:258-277: numerical failures still write the report, exit 1
template <class Body>
int guarded(Report& r, const std::string& path, Body&& body) {
  try {
    return body();
  } catch (const fgs::NumericalError& e) {
    r.status = "numerical-failure";
    r.diagnostic = e.what();
  } catch (const fgs::ResourceError& e) {
    r.status = "numerical-failure";
    r.diagnostic = e.what();
  }
  write_report(r, path);
  std::cerr << "numerical failure: " << r.diagnostic << '\n' << "report: " << path << '\n';
  return 1;
}

// ---- eigs (commands.cpp:339-358) -------------------------------------------
int run_eigs(Args& a) {
  CommonOpts o;
  io_flags(a, &o, true);
  kernel_flags(a, &o);
  fastsum_flags(a, &o);
  method_flags(a, &o);
  a.finish();
  Report rep;
  rep.command = "eigs";
  rep.method = o.method;
  rep.seed = o.seed;
  rep.parameters = echo_common(o);
  return guarded(rep, o.out, [&] {
    const PointCloud cloud = load_points_csv(o.in);
    const KernelSpec kernel = make_kernel(o);
    const FastsumParams params = make_params(o);
    const EigenPairs pairs = solve_pairs(cloud, kernel, params, o, &rep);
    if (o.with_reference) add_reference_metrics(cloud, kernel, pairs, o, &rep);
    return finish(rep, o.out,
                  "eigs: n=" + std::to_string(cloud.size()) + " k=" + std::to_string(pairs.count()) +
                      " lambda_1=" + std::to_string(pairs.count() ? pairs.values(0) : 0.0) + '\n');
  });
}

// ---- cluster (commands.cpp:362-391) ----------------------------------------
int run_cluster(Args& a) {
  CommonOpts o;
  io_flags(a, &o, true);
  kernel_flags(a, &o);
  fastsum_flags(a, &o);
  method_flags(a, &o);
  a.finish();
  Report rep;
  rep.command = "cluster";
  rep.method = o.method;
  rep.seed = o.seed;
  rep.parameters = echo_common(o);
  return guarded(rep, o.out, [&] {
    const PointCloud cloud = load_points_csv(o.in);
    const EigenPairs pairs = solve_pairs(cloud, make_kernel(o), make_params(o), o, &rep);
    fgs::KMeansOptions ko;
    ko.seed = o.seed;
    Timer t;
    const std::vector<int> labels = fgs::spectral_cluster(pairs, o.k, ko, o.device);
    rep.add_timing("cluster", t.seconds());
    save_labels_csv(labels, o.out + ".labels.csv");
    std::string summary = "cluster: n=" + std::to_string(cloud.size()) + " into " + std::to_string(o.k) + " groups\n";
    if (cloud.has_labels()) {
      const double rate = fgs::misclassification_rate_permuted(labels, cloud.labels);
      rep.add_metric("misclassification_rate_permuted", rate,
                     "fraction of points whose cluster disagrees with the input label, minimized over cluster "
                     "relabelings");
      summary += "misclassification (best relabeling): " + std::to_string(rate) + '\n';
    }
    return finish(rep, o.out, summary);
  });
}

// ---- bench (commands.cpp:722-845) ------------------------------------------
int run_bench(Args& a) {
  CommonOpts o;
  o.sigma = 3.5;
  std::vector<long long> sizes{8000, 16000, 32000, 64000};
  std::vector<std::string> methods{"nfft-lanczos"};
  int trials = 1, applies = 5;
  io_flags(a, &o, false);
  kernel_flags(a, &o);
  fastsum_flags(a, &o);
  a.get("k", &o.k);
  a.get("L", &o.sketch_l);
  a.get("M", &o.sketch_m);
  a.get("tol", &o.tol);
  a.get("with-reference", &o.with_reference);
  a.get_list("sizes", &sizes);
  a.get_list("methods", &methods);
  a.get("trials", &trials);
  a.get("applies", &applies);
  a.finish();
  Report rep;
  rep.command = "bench";
  rep.method = "sweep";
  rep.seed = o.seed;
  rep.parameters = echo_common(o);
  rep.parameters["sizes"] = sizes;
  rep.parameters["methods"] = methods;
  rep.parameters["trials"] = trials;
  for (const auto& m : methods)
    if (m != "nfft-lanczos" && m != "nystrom" && m != "nystrom-gauss-nfft" && m != "direct")
      throw fgs::ParameterError("unknown bench method " + m);
  return guarded(rep, o.out, [&] {
    const KernelSpec kernel = make_kernel(o);
    const FastsumParams params = make_params(o);
    Json cells = Json::array();
    std::string summary;
    std::vector<double> matvec_by_size;
    for (const auto& method : methods) {
      for (long long n : sizes) {
        if (n % 5 != 0) throw fgs::ParameterError("bench sizes must be divisible by the 5 spiral classes");
        std::vector<double> value_errors, residuals;
        double setup_s = 0.0, matvec_s = 0.0, solve_s = 0.0;
        for (int trial = 0; trial < trials; ++trial) {
          const std::uint64_t seed = o.seed + static_cast<std::uint64_t>(trial);
          const PointCloud cloud = gen_spiral(5, static_cast<int>(n / 5), 10.0, 2.0, seed);
          CommonOpts cell = o;
          cell.method = method;
          cell.seed = seed;
          Report sink;
          Timer setup;
          std::optional<AdjacencyOperator> op;
          op.emplace(cloud.coordinates, kernel, params,
                     method == "direct" ? AdjacencyBackend::Direct : (backend_of(method == "nystrom-gauss-nfft"
                                                                                      ? std::string("nfft-lanczos")
                                                                                      : method)),
                     o.device);
          setup_s += setup.seconds();
          {
            std::mt19937_64 rng(seed);
            std::normal_distribution<double> gauss;
            VectorXd x(n);
            for (Index i = 0; i < n; ++i) x(i) = gauss(rng);
            Timer mv;
            for (int r = 0; r < applies; ++r) x = op->apply_normalized(x);
            matvec_s += mv.seconds() / applies;
          }
          Timer solve;
          const EigenPairs pairs = solve_pairs(cloud, kernel, params, cell, &sink);
          solve_s += solve.seconds();
          if (o.with_reference && n <= kReferenceBudget) {
            AdjacencyOperator exact(cloud.coordinates, kernel, FastsumParams{}, AdjacencyBackend::Direct, o.device);
            residuals.push_back(fgs::max_residual(exact, pairs));
            value_errors.push_back(max_value_error(pairs, dense_reference_eig(exact, static_cast<int>(pairs.count()))));
          }
        }
        Json c = Json::object();
        c["method"] = method;
        c["n"] = n;
        c["trials"] = trials;
        c["setup_seconds"] = setup_s / trials;
        c["matvec_seconds"] = matvec_s / trials;
        c["solve_seconds"] = solve_s / trials;
        if (!value_errors.empty()) {
          auto stats = [](const std::vector<double>& v, const char* def) {
            double lo = v[0], hi = v[0], sum = 0.0;
            for (double x : v) {
              lo = std::min(lo, x);
              hi = std::max(hi, x);
              sum += x;
            }
            Json j = Json::object();
            j["min"] = lo;
            j["avg"] = sum / static_cast<double>(v.size());
            j["max"] = hi;
            j["definition"] = def;
            return j;
          };
          c["eigenvalue_error"] = stats(value_errors, "max_i |lambda_i - lambda_i^dense| per trial, aggregated");
          c["residual"] =
              stats(residuals, "max_i ||A v_i - lambda_i v_i||_2 with exact applies per trial, aggregated");
        }
        cells.push_back(c);
        if (method == methods.front()) matvec_by_size.push_back(matvec_s / trials);
        summary += method + " n=" + std::to_string(n) + ": matvec " + std::to_string(matvec_s / trials) +
                   " s, solve " + std::to_string(solve_s / trials) + " s\n";
      }
    }
    rep.extra["cells"] = cells;
    if (matvec_by_size.size() >= 2 && matvec_by_size.front() > 0.0)
      rep.add_metric("matvec_time_ratio", matvec_by_size.back() / matvec_by_size.front(),
                     "average fast matvec time at the largest size divided by the smallest size, first method");
    return finish(rep, o.out, summary);
  });
}

const char* kUsage =
    "fgs-b200: matrix-free spectral toolkit for fully connected kernel graphs (B200 build)\n"
    "usage: fgs-b200 <eigs|cluster|bench> [--options]\n";

int run(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage;
    return 2;
  }
  const std::string cmd = argv[1];
  if (cmd == "--help" || cmd == "-h") {
    std::cout << kUsage;
    return 0;
  }
  try {
    Args a(argc, argv, 2);
    if (cmd == "eigs") return run_eigs(a);
    if (cmd == "cluster") return run_cluster(a);
    if (cmd == "bench") return run_bench(a);
    if (cmd == "gen" || cmd == "segment" || cmd == "ssl-kernel" || cmd == "krr" || cmd == "ssl-pf")
      throw UsageError("command '" + cmd + "' is not part of the B200 build");
    throw UsageError("unknown command '" + cmd + "'");
  } catch (const UsageError& e) {  // CLI11::ParseError -> 2
    std::cerr << e.what() << '\n' << kUsage;
    return 2;
  } catch (const fgs::ParameterError& e) {
    std::cerr << "usage error: " << e.what() << '\n';
    return 2;
  } catch (const fgs::RangeError& e) {
    std::cerr << "usage error: " << e.what() << '\n';
    return 2;
  } catch (const fgs::ShapeError& e) {
    std::cerr << "usage error: " << e.what() << '\n';
    return 2;
  } catch (const FormatError& e) {
    std::cerr << "usage error: " << e.what() << '\n';
    return 2;
  } catch (const ParseError& e) {
    std::cerr << "input error: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}

}  // namespace cli

int main(int argc, char** argv) { return cli::run(argc, argv); }

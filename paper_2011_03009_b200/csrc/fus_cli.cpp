// `fus` command-line front end over the drop-in (namespace fus -> libfus.so -> libfusg.so):
// simulate / plan / converge / validate, with the reference's outputs and exit codes
// (reference: tools/fus_cli.cpp).  The reference parses options with CLI11 and writes the
// manifest with nlohmann::json, neither of which is in this image; both are replaced by small
// local equivalents with the same observable behaviour:
//   * options: `--name value` and `--name=value`; vector options take one or more values
//     (tools/fus_cli.cpp:271-306);
//   * manifest.json: nlohmann's dump(2) of a flat object: keys in sorted order, two-space
//     indent, shortest round-trip doubles with ".0" on integral values (tools/fus_cli.cpp:49-55,177);
//   * timings.csv: columns harmonic,n_voxels,meshing_s,interpolation_s,evaluate_Gk_s,compute_p_s
//     and the fixed-width console table (tools/fus_cli.cpp:113-131).
// Exit codes: 0 ok, 1 configuration error, 2 runtime error (tools/fus_cli.cpp:30-31).
#include <Eigen/Dense>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fus/analysis.hpp"
#include "fus/cascade.hpp"
#include "fus/io.hpp"
#include "fus/medium.hpp"
#include "fus/potential.hpp"
#include "fus/transducer.hpp"
#include "fus/vie.hpp"

namespace fs = std::filesystem;

namespace {

constexpr int kExitConfigError = 1;
constexpr int kExitRuntimeError = 2;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct RunConfig {  // tools/fus_cli.cpp:33-48
  std::string transducer = "H101";
  std::string medium = "water";
  double power = 100.0;
  double f0_override = 0.0;
  int n_harmonics = 5;
  int n_w = 6;
  double d = 10.2e-3;
  int n_points = 4096;
  std::string mode = "homogeneous";
  std::string medium_map;
  std::string out = "fus-out";
  int threads = 0;
  bool dump_fields = false;
  double width_scale = 1.0;
};

// ---------------------------------------------------------------- manifest (flat JSON object)
std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  // shortest round-trip significand, then nlohmann's layout (fixed for -4 < n <= 15, else d.ddde±XX)
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  const bool neg = s[0] == '-';
  if (neg) s.erase(0, 1);
  const auto epos = s.find('e');
  const int e10 = std::atoi(s.c_str() + epos + 1);
  std::string digits;
  for (std::size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits += s[i];
  const int len = int(digits.size());
  const int n = e10 + 1;  // position of the decimal point relative to the digit string
  std::string out;
  if (len <= n && n <= 15) {
    out = digits + std::string(n - len, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (len > 1) out += "." + digits.substr(1);
    const int k = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", k < 0 ? '-' : '+', std::abs(k));
    out += eb;
  }
  return (neg ? "-" : "") + out;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      case '\r': o += "\\r"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += c;
        }
    }
  }
  return o + "\"";
}

std::string manifest_json(const RunConfig& c) {
  std::map<std::string, std::string> kv;  // std::map: nlohmann's default object order
  kv["transducer"] = json_string(c.transducer);
  kv["medium"] = json_string(c.medium);
  kv["power"] = json_double(c.power);
  kv["f0_override"] = json_double(c.f0_override);
  kv["n_harmonics"] = std::to_string(c.n_harmonics);
  kv["n_w"] = std::to_string(c.n_w);
  kv["d"] = json_double(c.d);
  kv["n_points"] = std::to_string(c.n_points);
  kv["mode"] = json_string(c.mode);
  kv["medium_map"] = json_string(c.medium_map);
  kv["out"] = json_string(c.out);
  kv["threads"] = std::to_string(c.threads);
  kv["dump_fields"] = c.dump_fields ? "true" : "false";
  kv["width_scale"] = json_double(c.width_scale);
  std::string o = "{";
  bool first = true;
  for (const auto& [k, v] : kv) {
    o += first ? "\n" : ",\n";
    first = false;
    o += "  " + json_string(k) + ": " + v;
  }
  return o + "\n}";
}

// A flat JSON object of strings, numbers and booleans (what manifest_json writes).
std::map<std::string, std::string> parse_flat_json(const std::string& text, const std::string& path) {
  std::map<std::string, std::string> kv;
  std::size_t i = 0;
  auto fail = [&](const std::string& why) -> void {
    throw std::runtime_error("manifest '" + path + "': " + why + " at offset " + std::to_string(i));
  };
  auto ws = [&] {
    while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
  };
  auto str = [&]() -> std::string {
    if (i >= text.size() || text[i] != '"') fail("expected a string");
    ++i;
    std::string s;
    while (i < text.size() && text[i] != '"') {
      if (text[i] == '\\' && i + 1 < text.size()) {
        const char e = text[++i];
        if (e == 'n') s += '\n';
        else if (e == 't') s += '\t';
        else if (e == 'r') s += '\r';
        else if (e == 'u' && i + 4 < text.size()) {
          s += char(std::stoi(text.substr(i + 1, 4), nullptr, 16));
          i += 4;
        } else s += e;
        ++i;
      } else {
        s += text[i++];
      }
    }
    if (i >= text.size()) fail("unterminated string");
    ++i;
    return s;
  };
  ws();
  if (i >= text.size() || text[i] != '{') fail("expected '{'");
  ++i;
  ws();
  if (i < text.size() && text[i] == '}') return kv;
  for (;;) {
    ws();
    const std::string key = str();
    ws();
    if (i >= text.size() || text[i] != ':') fail("expected ':'");
    ++i;
    ws();
    if (i < text.size() && text[i] == '"') {
      kv[key] = str();
    } else {
      const std::size_t b = i;
      while (i < text.size() && text[i] != ',' && text[i] != '}' &&
             !std::isspace(static_cast<unsigned char>(text[i])))
        ++i;
      if (i == b) fail("expected a value");
      kv[key] = text.substr(b, i - b);
    }
    ws();
    if (i < text.size() && text[i] == ',') {
      ++i;
      continue;
    }
    if (i < text.size() && text[i] == '}') break;
    fail("expected ',' or '}'");
  }
  return kv;
}

RunConfig load_manifest(const std::string& path) {  // from_json, tools/fus_cli.cpp:57-72
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open manifest '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  const auto kv = parse_flat_json(ss.str(), path);
  auto at = [&](const char* k) -> const std::string& {
    const auto it = kv.find(k);
    if (it == kv.end()) throw std::runtime_error(std::string("manifest: missing key '") + k + "'");
    return it->second;
  };
  auto boolean = [&](const char* k) {
    const std::string& v = at(k);
    if (v == "true") return true;
    if (v == "false") return false;
    throw std::runtime_error(std::string("manifest: '") + k + "' is not a boolean");
  };
  RunConfig c;
  c.transducer = at("transducer");
  c.medium = at("medium");
  c.power = std::stod(at("power"));
  c.f0_override = std::stod(at("f0_override"));
  c.n_harmonics = std::stoi(at("n_harmonics"));
  c.n_w = std::stoi(at("n_w"));
  c.d = std::stod(at("d"));
  c.n_points = std::stoi(at("n_points"));
  c.mode = at("mode");
  c.medium_map = at("medium_map");
  c.out = at("out");
  c.threads = std::stoi(at("threads"));
  c.dump_fields = boolean("dump_fields");
  c.width_scale = std::stod(at("width_scale"));
  return c;
}

// ---------------------------------------------------------------- resolution (tools/fus_cli.cpp:86-111)
fus::Medium resolve_medium(const std::string& spec) {
  return fus::is_medium_preset(spec) ? fus::medium_preset(spec) : fus::load_medium(spec);
}

fus::BowlTransducer resolve_transducer(const RunConfig& cfg) {
  fus::BowlTransducer t = fus::is_transducer_preset(cfg.transducer)
                              ? fus::transducer_preset(cfg.transducer, cfg.power, cfg.n_points)
                              : fus::load_transducer(cfg.transducer, cfg.power);
  if (cfg.f0_override > 0.0) t.f0 = cfg.f0_override;
  return t;
}

fus::MediumMap resolve_medium_map(const RunConfig& cfg, const fus::Medium& background,
                                  const fus::VoxelGrid& grid) {
  if (cfg.medium_map.rfind("slab:", 0) == 0) {
    std::stringstream ss(cfg.medium_map.substr(5));
    std::string med, center, thickness;
    if (!std::getline(ss, med, ':') || !std::getline(ss, center, ':') || !std::getline(ss, thickness, ':'))
      throw std::invalid_argument("medium-map slab spec must be slab:<medium>:<center_m>:<thickness_m>");
    return fus::slab_map(grid, background, resolve_medium(med), std::stod(center), std::stod(thickness));
  }
  return fus::load_medium_map(cfg.medium_map, background);
}

// timings.csv + console table (tools/fus_cli.cpp:113-131)
void write_timing_table(const std::string& csv_path, const std::vector<fus::StageTiming>& rows) {
  std::vector<std::vector<double>> data;
  for (const auto& r : rows)
    data.push_back({double(r.harmonic), double(r.voxels), r.meshing_s, r.interpolation_s, r.kernel_s,
                    r.potential_s});
  fus::write_csv(csv_path,
                 {"harmonic", "n_voxels", "meshing_s", "interpolation_s", "evaluate_Gk_s", "compute_p_s"},
                 data);
  std::cout << std::left << std::setw(6) << "p_i" << std::setw(14) << "N voxels" << std::setw(12)
            << "Meshing" << std::setw(16) << "Interpolation" << std::setw(16) << "Evaluate G_ki"
            << std::setw(12) << "Compute p_i" << '\n';
  for (const auto& r : rows)
    std::cout << std::left << "p" << std::setw(5) << r.harmonic << std::setw(14) << double(r.voxels)
              << std::setw(12) << r.meshing_s << std::setw(16) << r.interpolation_s << std::setw(16)
              << r.kernel_s << std::setw(12) << r.potential_s << '\n';
}

// ---------------------------------------------------------------- subcommands
int cmd_simulate(const RunConfig& cfg) {  // tools/fus_cli.cpp:133-180
  const fus::Medium medium = resolve_medium(cfg.medium);
  const fus::BowlTransducer trans = resolve_transducer(cfg);
  if (cfg.mode != "homogeneous" && cfg.mode != "vie") throw ConfigError("--mode must be homogeneous or vie");
  if (cfg.n_harmonics < 1) throw ConfigError("--harmonics must be >= 1");

  fus::CascadeResult result;
  fus::MeshPlan plan;
  if (cfg.n_harmonics == 1) {
    const fus::DomainBox d2 = fus::reference_domain(trans, cfg.d);
    const fus::VoxelGrid grid = fus::make_grid(d2, medium.c0 / trans.f0 / cfg.n_w, 1, trans.focus());
    fus::SourceField src = fus::evaluate_source_field(trans, medium, grid);
    result.harmonics.push_back(std::move(src.field));
    result.source_normalization = src.normalization;
  } else {
    plan = fus::plan_nested_meshes(trans, medium, cfg.d, cfg.n_w, cfg.n_harmonics, cfg.width_scale);
    fus::CascadeConfig cc{medium, trans, plan, cfg.n_harmonics};
    if (cfg.mode == "vie") {
      if (cfg.medium_map.empty()) throw ConfigError("--mode vie requires --medium-map");
      const fus::MediumMap map = resolve_medium_map(cfg, medium, plan.for_harmonic(2).grid);
      result = fus::run_cascade_inhomogeneous(cc, map);
    } else {
      result = fus::run_cascade(cc);
    }
  }

  fs::create_directories(cfg.out);
  for (const auto& field : result.harmonics) {
    const int n = field.wavenumber.harmonic;
    const fus::OnAxisProfile prof = fus::extract_on_axis(field);
    fus::write_on_axis_csv(cfg.out + "/onaxis_p" + std::to_string(n) + ".csv", prof.x, prof.p);
    if (cfg.dump_fields) fus::write_field_dump(cfg.out + "/p" + std::to_string(n) + ".bin", field);
  }
  if (cfg.n_harmonics >= 2) {
    std::ofstream(cfg.out + "/meshplan.txt") << plan.report();
    write_timing_table(cfg.out + "/timings.csv", result.timings);
  }
  std::ofstream(cfg.out + "/manifest.json") << manifest_json(cfg) << '\n';
  std::cout << "wrote " << result.harmonics.size() << " harmonic(s) to " << cfg.out << '\n';
  return 0;
}

int cmd_plan(const RunConfig& cfg) {  // tools/fus_cli.cpp:182-189
  const fus::Medium medium = resolve_medium(cfg.medium);
  const fus::BowlTransducer trans = resolve_transducer(cfg);
  std::cout << fus::plan_nested_meshes(trans, medium, cfg.d, cfg.n_w, cfg.n_harmonics, cfg.width_scale).report();
  return 0;
}

int cmd_converge(const RunConfig& cfg, const std::string& study, const std::vector<int>& nw_values, int nw_ref,
                 double length, double width, const std::vector<double>& levels, bool q0_mode) {
  // tools/fus_cli.cpp:191-228
  const fus::Medium medium = resolve_medium(cfg.medium);
  const fus::BowlTransducer trans = resolve_transducer(cfg);
  std::vector<fus::ConvergenceRecord> records;
  if (study == "quadrature") {
    fus::DomainBox box;
    const Eigen::Vector3d focus = trans.focus();
    box.lo = {focus.x() - length / 2, -width / 2, -width / 2};
    box.hi = {focus.x() + length / 2, width / 2, width / 2};
    const fus::QuadratureStudy qs = fus::quadrature_convergence_study(trans, medium, box, nw_values, nw_ref);
    records = qs.records;
    std::cout << "fitted log-log slope: " << qs.slope << '\n';
  } else if (study == "domain") {
    const fus::MeshPlan plan = fus::plan_full_domain(trans, medium, cfg.d, cfg.n_w, cfg.n_harmonics, cfg.width_scale);
    fus::CascadeConfig cc{medium, trans, plan, cfg.n_harmonics};
    const fus::CascadeResult reference = fus::run_cascade(cc);
    records = fus::domain_shrink_study(cc, reference, levels, q0_mode);
  } else {
    throw ConfigError("--study must be quadrature or domain");
  }
  fs::create_directories(cfg.out);
  std::vector<std::vector<double>> rows;
  for (const auto& r : records) rows.push_back({double(r.harmonic), r.value, r.error_percent});
  const std::string control = records.empty() ? "value" : records.front().control;
  fus::write_csv(cfg.out + "/convergence.csv", {"harmonic", control, "error_percent"}, rows);
  for (const auto& r : records)
    std::cout << "p" << r.harmonic << "  " << r.control << " = " << r.value << "  error = " << r.error_percent
              << " %\n";
  return 0;
}

Eigen::VectorXcd random_vector(std::size_t n, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  Eigen::VectorXcd v(static_cast<Eigen::Index>(n));
  for (auto& x : v) {
    const double re = u(rng);
    const double im = u(rng);
    x = {re, im};
  }
  return v;
}

int cmd_validate() {  // the built-in invariant suite, tools/fus_cli.cpp:230-264
  int failures = 0;
  auto check = [&](const std::string& name, bool ok) {
    std::cout << (ok ? "[ ok ] " : "[FAIL] ") << name << '\n';
    if (!ok) ++failures;
  };
  const fus::Medium water = fus::medium_preset("water");
  const fus::Wavenumber k1 = fus::complex_wavenumber(water, 1.1e6, 1);
  const fus::Wavenumber k3 = fus::complex_wavenumber(water, 1.1e6, 3);
  check("Re(k_n) = n Re(k_1)", std::abs(k3.k.real() - 3 * k1.k.real()) < 1e-9 * k3.k.real());
  check("Im(k_n)/Im(k_1) = n^eta", std::abs(k3.k.imag() / k1.k.imag() - std::pow(3.0, water.eta)) < 1e-9);

  const auto pts = fus::distribute_points(35e-3, 16.5e-3, 512);
  bool on_sphere = pts.size() == 512;
  for (const auto& p : pts) on_sphere = on_sphere && std::abs((p - Eigen::Vector3d(35e-3, 0, 0)).norm() - 35e-3) < 1e-12;
  check("cap points on the focal sphere", on_sphere);

  fus::DomainBox box{{0, 0, 0}, {8e-3, 7e-3, 6e-3}};
  const fus::VoxelGrid grid = fus::make_grid(box, 1e-3, 2);
  // the reference draws Eigen::VectorXcd::Random; any bounded source exercises the same check
  const Eigen::VectorXcd f = random_vector(grid.count(), 2011);
  const fus::GreenKernel kernel(grid, k1);
  const Eigen::VectorXcd u_fft = kernel.apply(f);
  const Eigen::VectorXcd u_dir = fus::direct_potential_oracle(k1, grid, f);
  Eigen::VectorXcd diff = u_fft;
  for (Eigen::Index i = 0; i < diff.size(); ++i) diff[i] -= u_dir[i];
  check("FFT convolution matches direct summation", diff.cwiseAbs().maxCoeff() < 1e-12 * u_dir.cwiseAbs().maxCoeff());

  fus::HarmonicField hf{grid, Eigen::VectorXcd::Constant(grid.count(), 2.5), k1};
  const fus::HarmonicField hi = fus::interpolate(hf, grid);
  double worst = 0.0;
  for (Eigen::Index i = 0; i < hi.values.size(); ++i) worst = std::max(worst, std::abs(hi.values[i] - hf.values[i]));
  check("interpolation is the identity on the same grid", worst == 0.0);

  std::cout << (failures == 0 ? "all checks passed\n" : "some checks FAILED\n");
  return failures == 0 ? 0 : kExitRuntimeError;
}

// ---------------------------------------------------------------- option parsing
struct Args {
  std::vector<std::string> v;
  std::size_t i = 0;
};

double to_double(const std::string& opt, const std::string& s) {
  try {
    std::size_t n = 0;
    const double x = std::stod(s, &n);
    if (n == s.size()) return x;
  } catch (const std::exception&) {
  }
  throw ConfigError(opt + ": '" + s + "' is not a number");
}

int to_int(const std::string& opt, const std::string& s) {
  try {
    std::size_t n = 0;
    const long x = std::stol(s, &n);
    if (n == s.size() && x >= INT32_MIN && x <= INT32_MAX) return int(x);
  } catch (const std::exception&) {
  }
  throw ConfigError(opt + ": '" + s + "' is not an integer");
}

void usage(std::ostream& o) {
  o << "Weakly nonlinear focused-ultrasound harmonics via FFT volume potentials\n"
       "usage: fus {simulate|plan|converge|validate} [options]\n"
       "common: --transducer --medium --power --f0 --harmonics --nw --d --np --width-scale --out --threads\n"
       "simulate: --mode homogeneous|vie --medium-map <hdr|slab:med:center:thickness> --dump-fields --manifest <json>\n"
       "converge: --study quadrature|domain --nw-list <n...> --nw-ref --length --width --levels <x...> --q0\n";
}

}  // namespace

int main(int argc, char** argv) {
  RunConfig cfg;
  std::string manifest_path, study = "quadrature";
  std::vector<int> nw_values{4, 6, 8, 10};
  int nw_ref = 20;
  double length = 20e-3, width = 4e-3;
  std::vector<double> levels{1.0, 0.8, 0.6, 0.4, 0.2};
  bool q0_mode = false;
  std::string sub;
  try {
    if (argc < 2) throw ConfigError("a subcommand is required (simulate, plan, converge, validate)");
    sub = argv[1];
    if (sub == "-h" || sub == "--help") {
      usage(std::cout);
      return 0;
    }
    if (sub != "simulate" && sub != "plan" && sub != "converge" && sub != "validate")
      throw ConfigError("unknown subcommand '" + sub + "'");
    std::vector<std::string> a(argv + 2, argv + argc);
    for (std::size_t i = 0; i < a.size(); ++i) {
      std::string opt = a[i], val;
      bool has_inline = false;
      if (const auto eq = opt.find('='); opt.rfind("--", 0) == 0 && eq != std::string::npos) {
        val = opt.substr(eq + 1);
        opt = opt.substr(0, eq);
        has_inline = true;
      }
      auto next = [&]() -> std::string {
        if (has_inline) return val;
        if (i + 1 >= a.size()) throw ConfigError(opt + " requires a value");
        return a[++i];
      };
      auto many = [&]() -> std::vector<std::string> {
        std::vector<std::string> out;
        if (has_inline) {
          out.push_back(val);
        }
        while (i + 1 < a.size() && a[i + 1].rfind("--", 0) != 0) out.push_back(a[++i]);
        if (out.empty()) throw ConfigError(opt + " requires at least one value");
        return out;
      };
      if (opt == "-h" || opt == "--help") {
        usage(std::cout);
        return 0;
      } else if (sub == "validate") {
        throw ConfigError("validate takes no options (got '" + opt + "')");
      } else if (opt == "--transducer") cfg.transducer = next();
      else if (opt == "--medium") cfg.medium = next();
      else if (opt == "--power") cfg.power = to_double(opt, next());
      else if (opt == "--f0") cfg.f0_override = to_double(opt, next());
      else if (opt == "--harmonics") cfg.n_harmonics = to_int(opt, next());
      else if (opt == "--nw") cfg.n_w = to_int(opt, next());
      else if (opt == "--d") cfg.d = to_double(opt, next());
      else if (opt == "--np") cfg.n_points = to_int(opt, next());
      else if (opt == "--width-scale") cfg.width_scale = to_double(opt, next());
      else if (opt == "--out") cfg.out = next();
      else if (opt == "--threads") cfg.threads = to_int(opt, next());
      else if (sub == "simulate" && opt == "--mode") cfg.mode = next();
      else if (sub == "simulate" && opt == "--medium-map") cfg.medium_map = next();
      else if (sub == "simulate" && opt == "--dump-fields") cfg.dump_fields = true;
      else if (sub == "simulate" && opt == "--manifest") manifest_path = next();
      else if (sub == "converge" && opt == "--study") study = next();
      else if (sub == "converge" && opt == "--nw-list") {
        nw_values.clear();
        for (const auto& s : many()) nw_values.push_back(to_int(opt, s));
      } else if (sub == "converge" && opt == "--nw-ref") nw_ref = to_int(opt, next());
      else if (sub == "converge" && opt == "--length") length = to_double(opt, next());
      else if (sub == "converge" && opt == "--width") width = to_double(opt, next());
      else if (sub == "converge" && opt == "--levels") {
        levels.clear();
        for (const auto& s : many()) levels.push_back(to_double(opt, s));
      } else if (sub == "converge" && opt == "--q0") q0_mode = true;
      else throw ConfigError("unknown option '" + opt + "' for " + sub);
    }
  } catch (const ConfigError& e) {
    std::cerr << "config error: " << e.what() << '\n';
    usage(std::cerr);
    return kExitConfigError;
  }

  try {
    if (!manifest_path.empty()) cfg = load_manifest(manifest_path);
    // threads: the reference sets the OpenMP team size; the device path has no host team, so
    // the value is only recorded in the manifest.
    if (sub == "simulate") return cmd_simulate(cfg);
    if (sub == "plan") return cmd_plan(cfg);
    if (sub == "converge") return cmd_converge(cfg, study, nw_values, nw_ref, length, width, levels, q0_mode);
    return cmd_validate();
  } catch (const ConfigError& e) {
    std::cerr << "config error: " << e.what() << '\n';
    return kExitConfigError;
  } catch (const std::invalid_argument& e) {
    std::cerr << "config error: " << e.what() << '\n';
    return kExitConfigError;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitRuntimeError;
  }
}

// namespace fus file formats (reference include/fus/io.hpp): host code with the reference's
// file contracts (src/io.cpp) -- written here from those contracts.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>

#include "fus/grid.hpp"
#include "fus/io.hpp"
#include "fus/medium.hpp"
#include "fus/transducer.hpp"
#include "fus/vie.hpp"

namespace fus {
namespace {

std::string strip(const std::string& s) {
  std::size_t b = 0, e = s.size();
  while (b < e && (s[b] == ' ' || s[b] == '\t' || s[b] == '\r')) ++b;
  while (e > b && (s[e - 1] == ' ' || s[e - 1] == '\t' || s[e - 1] == '\r')) --e;
  return s.substr(b, e - b);
}

// %.17g: the stream format the reference writes (std::setprecision(17), general notation)
std::string num(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

std::ofstream open_out(const std::string& path, std::ios::openmode mode = std::ios::out) {
  std::ofstream out(path, mode);
  if (!out) throw std::runtime_error("cannot write '" + path + "'");
  return out;
}

}  // namespace

std::map<std::string, std::string> parse_key_value_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open config file '" + path + "'");
  std::map<std::string, std::string> kv;
  std::string line;
  for (int n = 1; std::getline(in, line); ++n) {
    const std::string t = strip(line);
    if (t.empty() || t[0] == '#') continue;
    const std::size_t eq = t.find('=');
    const std::string where = path + ":" + std::to_string(n) + ": ";
    if (eq == std::string::npos) throw std::runtime_error(where + "expected 'key = value'");
    const std::string key = strip(t.substr(0, eq));
    if (key.empty()) throw std::runtime_error(where + "empty key");
    kv[key] = strip(t.substr(eq + 1));
  }
  return kv;
}

double require_double(const std::map<std::string, std::string>& kv, const std::string& key,
                      const std::string& context) {
  const std::string& s = require_string(kv, key, context);
  std::size_t used = 0;
  double v = 0.0;
  try {
    v = std::stod(s, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != s.size())
    throw std::runtime_error(context + ": key '" + key + "' is not a number: '" + s + "'");
  return v;
}

std::string require_string(const std::map<std::string, std::string>& kv, const std::string& key,
                           const std::string& context) {
  const auto it = kv.find(key);
  if (it == kv.end()) throw std::runtime_error(context + ": missing required key '" + key + "'");
  return it->second;
}

void write_on_axis_csv(const std::string& path, const Eigen::VectorXd& x, const Eigen::VectorXcd& p) {
  std::ofstream out = open_out(path);
  out << "x_m,re_Pa,im_Pa,abs_Pa\n";
  for (Eigen::Index i = 0; i < x.size(); ++i)
    out << num(x[i]) << ',' << num(p[i].real()) << ',' << num(p[i].imag()) << ',' << num(std::abs(p[i])) << '\n';
}

void write_field_dump(const std::string& path, const HarmonicField& field) {
  {
    std::ofstream out = open_out(path, std::ios::binary);
    out.write(reinterpret_cast<const char*>(field.values.data()),
              std::streamsize(field.values.size() * Eigen::Index(sizeof(std::complex<double>))));
  }
  std::ofstream hdr = open_out(path + ".hdr");
  const VoxelGrid& g = field.grid;
  hdr << "nx = " << g.dims.x() << "\nny = " << g.dims.y() << "\nnz = " << g.dims.z() << "\ndx = " << num(g.dx)
      << "\norigin_x = " << num(g.box.lo.x()) << "\norigin_y = " << num(g.box.lo.y())
      << "\norigin_z = " << num(g.box.lo.z()) << "\nharmonic = " << field.wavenumber.harmonic
      << "\nk_re = " << num(field.wavenumber.k.real()) << "\nk_im = " << num(field.wavenumber.k.imag())
      << "\nlayout = x_fastest_complex_f64_le\n";
}

void write_csv(const std::string& path, const std::vector<std::string>& columns,
               const std::vector<std::vector<double>>& rows) {
  std::ofstream out = open_out(path);
  for (std::size_t i = 0; i < columns.size(); ++i) out << columns[i] << (i + 1 < columns.size() ? ',' : '\n');
  for (const auto& row : rows)
    for (std::size_t i = 0; i < row.size(); ++i) out << num(row[i]) << (i + 1 < row.size() ? ',' : '\n');
}

// medium-map rasters (include/fus/vie.hpp:42-46; src/vie.cpp:83-131): a key = value header
// (nx, ny, nz, dx, origin_*, raster) and little-endian (c, beta) double pairs, x fastest
MediumMap load_medium_map(const std::string& header_path, const Medium& background) {
  const auto kv = parse_key_value_file(header_path);
  VoxelGrid g;
  g.dims = {int(require_double(kv, "nx", header_path)), int(require_double(kv, "ny", header_path)),
            int(require_double(kv, "nz", header_path))};
  g.dx = require_double(kv, "dx", header_path);
  g.box.lo = {require_double(kv, "origin_x", header_path), require_double(kv, "origin_y", header_path),
              require_double(kv, "origin_z", header_path)};
  for (int a = 0; a < 3; ++a) g.box.hi[a] = g.box.lo[a] + g.dims[a] * g.dx;
  const std::string name = require_string(kv, "raster", header_path);
  const std::size_t slash = header_path.find_last_of('/');
  const std::string raster = (slash == std::string::npos ? std::string() : header_path.substr(0, slash + 1)) + name;
  std::ifstream in(raster, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open medium-map raster '" + raster + "'");
  MediumMap m;
  m.grid = g;
  m.background = background;
  m.c.resize(Eigen::Index(g.count()));
  m.beta.resize(Eigen::Index(g.count()));
  for (std::size_t i = 0; i < g.count(); ++i) {
    double pair[2];
    if (!in.read(reinterpret_cast<char*>(pair), sizeof(pair)))
      throw std::runtime_error("medium-map raster '" + raster + "' is truncated");
    m.c[Eigen::Index(i)] = pair[0];
    m.beta[Eigen::Index(i)] = pair[1];
  }
  return m;
}

void write_medium_map(const std::string& header_path, const std::string& raster_path, const MediumMap& map) {
  {
    std::ofstream hdr = open_out(header_path);
    const std::size_t slash = raster_path.find_last_of('/');
    hdr << "nx = " << map.grid.dims.x() << "\nny = " << map.grid.dims.y() << "\nnz = " << map.grid.dims.z()
        << "\ndx = " << num(map.grid.dx) << "\norigin_x = " << num(map.grid.box.lo.x())
        << "\norigin_y = " << num(map.grid.box.lo.y()) << "\norigin_z = " << num(map.grid.box.lo.z())
        << "\nraster = " << (slash == std::string::npos ? raster_path : raster_path.substr(slash + 1)) << "\n";
  }
  std::ofstream out = open_out(raster_path, std::ios::binary);
  for (Eigen::Index i = 0; i < map.c.size(); ++i) {
    const double pair[2] = {map.c[i], map.beta[i]};
    out.write(reinterpret_cast<const char*>(pair), sizeof(pair));
  }
}

// Medium / transducer config files (src/medium.cpp:58-69, src/transducer.cpp:94-102): the same
// keys, the same missing-key and malformed-number errors (require_*), and the medium's
// validation warnings on stderr.
Medium load_medium(const std::string& path) {
  const auto kv = parse_key_value_file(path);
  Medium m;
  m.name = require_string(kv, "name", path);
  m.rho0 = require_double(kv, "rho0", path);
  m.c0 = require_double(kv, "c0", path);
  m.beta = require_double(kv, "beta", path);
  m.alpha0 = require_double(kv, "alpha0", path);
  m.eta = require_double(kv, "eta", path);
  for (const auto& w : m.validate()) std::cerr << "warning: " << w << "\n";
  return m;
}

BowlTransducer load_transducer(const std::string& path, double power) {
  const auto kv = parse_key_value_file(path);
  const std::string name = require_string(kv, "name", path);
  const double f0 = require_double(kv, "f0", path);
  const double l = require_double(kv, "focal_length", path);
  const double R = require_double(kv, "outer_radius", path);
  const int n_points = int(require_double(kv, "n_points", path));
  return make_bowl(name, f0, l, R, power, n_points);
}

}  // namespace fus

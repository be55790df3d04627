// tenrec_b200_cli — the reference's `tenrec` front end (proj/tools/cli.cpp) for
// the subcommands on and around the PASD hot path, over the C++ drop-in
// (include/tenrec_b200/pasd.hpp) and the C-ABI (include/pasd_b200.h):
//
//   synth    --dims --rank|--ranks [--corruption --seed --mode additive|replace255] --out-prefix
//            (cli.cpp:158-208; generator on the device, pasd_b200_synth)
//   recover  --input | --from-manifest, --out-prefix, [--truth --strict --no-z --solver pasd|snn
//            --lambdas --ranks --target-rank --alphas --mu0 --mu-max --mu-growth --eps --maxiter]
//            (cli.cpp:95-130, 210-354)
//   certify  --manifest [--truth]   (cli.cpp:452-553; nuclear norms on the device)
//   defaults                        (cli.cpp:557-567)
//
// Files: TNSR tensors (io.cpp:85-169) and key = value manifests (io.cpp:258-407),
// both written atomically (temp file + rename, io.cpp:31-68).  Exit codes of
// cli.hpp:9-14: 0 ok, 1 usage / argument, 2 I/O, 3 numerical / failed check,
// 4 non-convergence with --strict.  CLI11 (the reference's parser, absent
// here) is replaced by a small `--key value` / `--key=value` parser.
//
//   g++ -std=c++17 -O2 -Iinclude tools/tenrec_b200_cli.cpp -Lpaper_1712_09999_b200 -lpasd_b200
//       -Wl,-rpath,$PWD/paper_1712_09999_b200 -o tenrec_b200
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "tenrec_b200/pasd.hpp"

using namespace tenrec_b200;
namespace fs = std::filesystem;

namespace {

constexpr double kDefaultMu0 = 1e-4, kDefaultMuMax = 1e10, kDefaultMuGrowth = 1.1, kDefaultEps = 1e-5;
constexpr int kDefaultMaxiter = 1000;  // cli.cpp:27-31

std::string format_double(double v) {  // io.cpp:171-175
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

// ------------------------------------------------------------------ files
class AtomicFile {  // io.cpp:31-68
 public:
  explicit AtomicFile(const fs::path& p) : target_(p) {
    static unsigned counter = 0;
    temp_ = p;
    temp_ += ".tmp" + std::to_string((unsigned long)::getpid()) + "." + std::to_string(counter++);
    out_.open(temp_, std::ios::binary | std::ios::trunc);
    if (!out_) throw IoError("cannot open '" + temp_.string() + "' for writing");
  }
  ~AtomicFile() {
    if (!done_) {
      out_.close();
      std::error_code ec;
      fs::remove(temp_, ec);
    }
  }
  std::ostream& stream() { return out_; }
  void commit() {
    out_.flush();
    if (!out_) throw IoError("write to '" + temp_.string() + "' failed");
    out_.close();
    std::error_code ec;
    fs::rename(temp_, target_, ec);
    if (ec) throw IoError("cannot rename '" + temp_.string() + "' to '" + target_.string() + "': " + ec.message());
    done_ = true;
  }

 private:
  fs::path target_, temp_;
  std::ofstream out_;
  bool done_ = false;
};

void put_u16(std::ostream& o, uint16_t v) {
  const unsigned char b[2] = {(unsigned char)(v & 0xff), (unsigned char)(v >> 8)};
  o.write(reinterpret_cast<const char*>(b), 2);
}
void put_u64(std::ostream& o, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)((v >> (8 * i)) & 0xff);
  o.write(reinterpret_cast<const char*>(b), 8);
}

DenseTensor read_tensor(const fs::path& path) {  // io.cpp:85-149, same checks and messages
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open '" + path.string() + "' for reading");
  auto read_exact = [&](char* dst, std::streamsize n, uint64_t off, const char* what) {
    in.read(dst, n);
    if (in.gcount() != n)
      throw IoError("'" + path.string() + "': truncated " + what + " at byte offset " +
                    std::to_string(off + (uint64_t)in.gcount()) + " (needed " + std::to_string(n) + " bytes, got " +
                    std::to_string(in.gcount()) + ")");
  };
  char magic[4];
  read_exact(magic, 4, 0, "magic");
  if (std::memcmp(magic, "TNSR", 4) != 0)
    throw IoError("'" + path.string() + "': bad magic at byte offset 0 (expected \"TNSR\")");
  unsigned char hdr[4];
  read_exact(reinterpret_cast<char*>(hdr), 4, 4, "header");
  const uint16_t version = (uint16_t)(hdr[0] | (hdr[1] << 8)), order = (uint16_t)(hdr[2] | (hdr[3] << 8));
  if (version != 1) throw IoError("'" + path.string() + "': unsupported version " + std::to_string(version) +
                                  " at byte offset 4");
  if (order == 0) throw IoError("'" + path.string() + "': zero order at byte offset 6");
  std::vector<Index> dims(order);
  for (uint16_t n = 0; n < order; ++n) {
    unsigned char raw[8];
    read_exact(reinterpret_cast<char*>(raw), 8, 8 + 8ull * n, "dimension");
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)raw[i] << (8 * i);
    if (v == 0 || v > (uint64_t)std::numeric_limits<Index>::max())
      throw IoError("'" + path.string() + "': invalid dimension " + std::to_string(v) + " at byte offset " +
                    std::to_string(8 + 8ull * n));
    dims[n] = (Index)v;
  }
  Index total = 1;
  for (Index d : dims) {
    if (total > std::numeric_limits<Index>::max() / d) throw ArgumentError("dimension product overflows");
    total *= d;
  }
  const uint64_t payload = 8 + 8ull * order;
  std::vector<double> data((size_t)total);
  in.read(reinterpret_cast<char*>(data.data()), (std::streamsize)(sizeof(double) * data.size()));
  const auto got = in.gcount();
  if (got != (std::streamsize)(sizeof(double) * data.size()))
    throw IoError("'" + path.string() + "': truncated payload at byte offset " + std::to_string(payload + (uint64_t)got) +
                  " (expected " + std::to_string(sizeof(double) * data.size()) + " payload bytes, got " +
                  std::to_string(got) + ")");
  if (in.peek() != std::ifstream::traits_type::eof())
    throw IoError("'" + path.string() + "': trailing bytes after payload at byte offset " +
                  std::to_string(payload + sizeof(double) * data.size()));
  for (size_t i = 0; i < data.size(); ++i)
    if (!std::isfinite(data[i]))
      throw IoError("'" + path.string() + "': non-finite value at payload index " + std::to_string(i) +
                    " (byte offset " + std::to_string(payload + sizeof(double) * i) + ")");
  return DenseTensor::from_data(std::move(dims), std::move(data));
}

void ensure_parent_dir(const fs::path& p) {
  if (!p.parent_path().empty()) fs::create_directories(p.parent_path());
}

void write_tensor(const DenseTensor& t, const fs::path& path) {  // io.cpp:151-169
  if (t.order() < 1) throw ArgumentError("write_tensor: empty tensor");
  for (Index i = 0; i < t.size(); ++i)
    if (!std::isfinite(t[i])) throw ArgumentError("write_tensor: tensor contains non-finite entries");
  AtomicFile f(path);
  std::ostream& o = f.stream();
  o.write("TNSR", 4);
  put_u16(o, 1);
  put_u16(o, (uint16_t)t.order());
  for (Index d : t.dims()) put_u64(o, (uint64_t)d);
  o.write(reinterpret_cast<const char*>(t.data()), (std::streamsize)(sizeof(double) * (size_t)t.size()));
  f.commit();
}

uint64_t tensor_checksum(const DenseTensor& t) {  // FNV-1a over order, dims, payload (bench.cpp:293-310)
  uint64_t h = 0xcbf29ce484222325ULL;
  auto mix = [&h](const unsigned char* b, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      h ^= b[i];
      h *= 0x100000001b3ULL;
    }
  };
  const uint64_t order = (uint64_t)t.order();
  mix(reinterpret_cast<const unsigned char*>(&order), 8);
  for (Index d : t.dims()) {
    const uint64_t v = (uint64_t)d;
    mix(reinterpret_cast<const unsigned char*>(&v), 8);
  }
  mix(reinterpret_cast<const unsigned char*>(t.data()), (size_t)t.size() * sizeof(double));
  return h;
}
std::string checksum_hex(uint64_t v) {
  char buf[17];
  std::snprintf(buf, sizeof(buf), "%016llx", (unsigned long long)v);
  return buf;
}

class Manifest {  // RunManifest, io.cpp:258-407
 public:
  void set(const std::string& k, std::string v) {
    for (auto& e : entries_)
      if (e.first == k) {
        e.second = std::move(v);
        return;
      }
    entries_.emplace_back(k, std::move(v));
  }
  void set_double(const std::string& k, double v) { set(k, format_double(v)); }
  void set_int(const std::string& k, long long v) { set(k, std::to_string(v)); }
  void set_bool(const std::string& k, bool v) { set(k, v ? "true" : "false"); }
  void set_doubles(const std::string& k, const std::vector<double>& v) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + format_double(v[i]);
    set(k, s);
  }
  void set_indices(const std::string& k, const std::vector<Index>& v) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    set(k, s);
  }
  bool has(const std::string& k) const {
    for (const auto& e : entries_)
      if (e.first == k) return true;
    return false;
  }
  const std::string& get(const std::string& k) const {
    for (const auto& e : entries_)
      if (e.first == k) return e.second;
    throw IoError("manifest: missing key '" + k + "'");
  }
  double get_double(const std::string& k) const {
    const std::string& raw = get(k);
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(raw.c_str(), &end);
    if (end == raw.c_str() || *end != '\0' || errno == ERANGE)
      throw IoError("manifest: key '" + k + "' is not a number: '" + raw + "'");
    return v;
  }
  long long get_int(const std::string& k) const {
    const std::string& raw = get(k);
    char* end = nullptr;
    errno = 0;
    const long long v = std::strtoll(raw.c_str(), &end, 10);
    if (end == raw.c_str() || *end != '\0' || errno == ERANGE)
      throw IoError("manifest: key '" + k + "' is not an integer: '" + raw + "'");
    return v;
  }
  std::vector<std::string> split(const std::string& k) const {
    std::vector<std::string> parts;
    std::string cur;
    const std::string& raw = get(k);
    for (char c : raw) {
      if (c == ',') {
        parts.push_back(cur);
        cur.clear();
      } else {
        cur += c;
      }
    }
    if (!raw.empty()) parts.push_back(cur);
    return parts;
  }
  std::vector<double> get_doubles(const std::string& k) const {
    std::vector<double> out;
    for (const std::string& p : split(k)) {
      char* end = nullptr;
      out.push_back(std::strtod(p.c_str(), &end));
      if (end == p.c_str() || *end != '\0')
        throw IoError("manifest: key '" + k + "' has a malformed number: '" + p + "'");
    }
    return out;
  }
  std::vector<Index> get_indices(const std::string& k) const {
    std::vector<Index> out;
    for (const std::string& p : split(k)) {
      char* end = nullptr;
      out.push_back((Index)std::strtoll(p.c_str(), &end, 10));
      if (end == p.c_str() || *end != '\0')
        throw IoError("manifest: key '" + k + "' has a malformed integer: '" + p + "'");
    }
    return out;
  }
  void save(const fs::path& p) const {
    AtomicFile f(p);
    for (const auto& [k, v] : entries_) f.stream() << k << " = " << v << '\n';
    f.commit();
  }
  static Manifest load(const fs::path& p) {
    std::ifstream in(p);
    if (!in) throw IoError("cannot open manifest '" + p.string() + "'");
    Manifest m;
    std::string line;
    size_t lineno = 0;
    auto trim = [](std::string s) {
      const auto a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
      return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
    };
    while (std::getline(in, line)) {
      ++lineno;
      if (line.empty() || line[0] == '#') continue;
      const auto pos = line.find('=');
      if (pos == std::string::npos)
        throw IoError("manifest '" + p.string() + "': malformed line " + std::to_string(lineno));
      m.set(trim(line.substr(0, pos)), trim(line.substr(pos + 1)));
    }
    return m;
  }

 private:
  std::vector<std::pair<std::string, std::string>> entries_;
};

// ------------------------------------------------------------------ arguments
struct Args {
  std::map<std::string, std::string> opt;
  std::map<std::string, bool> flag;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string str(const std::string& k, const std::string& d = "") const { return has(k) ? opt.at(k) : d; }
};

Args parse(const std::vector<std::string>& argv, const std::vector<std::string>& options,
           const std::vector<std::string>& flags) {
  Args a;
  for (size_t i = 0; i < argv.size(); ++i) {
    std::string k = argv[i], v;
    const auto eq = k.find('=');
    if (eq != std::string::npos) {
      v = k.substr(eq + 1);
      k = k.substr(0, eq);
    }
    if (std::find(flags.begin(), flags.end(), k) != flags.end()) {
      a.flag[k] = true;
      continue;
    }
    if (std::find(options.begin(), options.end(), k) == options.end())
      throw ArgumentError("unknown option '" + k + "'");
    if (eq == std::string::npos) {
      if (i + 1 >= argv.size()) throw ArgumentError("option " + k + " needs a value");
      v = argv[++i];
    }
    a.opt[k] = v;
  }
  return a;
}

double to_double(const std::string& s, const std::string& what) {
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (end == s.c_str() || *end != '\0') throw ArgumentError("malformed value '" + s + "' for " + what);
  return v;
}
long long to_int(const std::string& s, const std::string& what) {
  char* end = nullptr;
  const long long v = std::strtoll(s.c_str(), &end, 10);
  if (end == s.c_str() || *end != '\0') throw ArgumentError("malformed value '" + s + "' for " + what);
  return v;
}
std::vector<double> to_doubles(const std::string& s, const std::string& what) {
  std::vector<double> out;
  std::stringstream ss(s);
  std::string p;
  while (std::getline(ss, p, ',')) out.push_back(to_double(p, what));
  return out;
}
std::vector<Index> to_indices(const std::string& s, const std::string& what) {
  std::vector<Index> out;
  std::stringstream ss(s);
  std::string p;
  while (std::getline(ss, p, ',')) out.push_back((Index)to_int(p, what));
  return out;
}

// ------------------------------------------------------------------ solver options (cli.cpp:83-130)
struct SolverOptions {
  std::string solver = "pasd";
  std::vector<double> lambdas, alphas;
  std::vector<Index> ranks;
  Index target_rank = 0;
  double mu0 = kDefaultMu0, mu_max = kDefaultMuMax, mu_growth = kDefaultMuGrowth, eps = kDefaultEps;
  int maxiter = kDefaultMaxiter;
};
const std::vector<std::string> kSolverOpts = {"--solver", "--lambdas", "--ranks",     "--target-rank", "--alphas",
                                              "--mu0",    "--mu-max",  "--mu-growth", "--eps",         "--maxiter",
                                              "--rpca-lambda"};

SolverOptions solver_options(const Args& a) {
  SolverOptions o;
  o.solver = a.str("--solver", "pasd");
  if (o.solver != "pasd" && o.solver != "snn" && o.solver != "rpca")
    throw ArgumentError("--solver: " + o.solver + " not in {pasd, snn, rpca}");
  if (a.has("--lambdas")) o.lambdas = to_doubles(a.str("--lambdas"), "--lambdas");
  if (a.has("--ranks")) o.ranks = to_indices(a.str("--ranks"), "--ranks");
  if (a.has("--target-rank")) o.target_rank = (Index)to_int(a.str("--target-rank"), "--target-rank");
  if (a.has("--alphas")) o.alphas = to_doubles(a.str("--alphas"), "--alphas");
  if (a.has("--mu0")) o.mu0 = to_double(a.str("--mu0"), "--mu0");
  if (a.has("--mu-max")) o.mu_max = to_double(a.str("--mu-max"), "--mu-max");
  if (a.has("--mu-growth")) o.mu_growth = to_double(a.str("--mu-growth"), "--mu-growth");
  if (a.has("--eps")) o.eps = to_double(a.str("--eps"), "--eps");
  if (a.has("--maxiter")) o.maxiter = (int)to_int(a.str("--maxiter"), "--maxiter");
  return o;
}

PasdConfig build_pasd_config(const SolverOptions& o, const std::vector<Index>& dims) {  // cli.cpp:112-130
  PasdConfig cfg;
  cfg.lambdas = o.lambdas.empty() ? PasdConfig::default_lambdas(dims) : o.lambdas;
  if (!o.ranks.empty())
    cfg.ranks = o.ranks;
  else if (o.target_rank > 0)
    cfg.ranks.assign(dims.size(), PasdConfig::default_rank_bound(o.target_rank));
  else
    throw ArgumentError("pasd needs --ranks or --target-rank");
  cfg.mu0 = o.mu0;
  cfg.mu_max = o.mu_max;
  cfg.rho = o.mu_growth;
  cfg.eps = o.eps;
  cfg.maxiter = o.maxiter;
  cfg.output_weights = o.alphas;
  cfg.validate(dims);
  return cfg;
}

SnnConfig build_snn_config(const SolverOptions& o, const std::vector<Index>& dims) {  // cli.cpp:132-143
  SnnConfig cfg;
  cfg.lambdas = o.lambdas.empty() ? PasdConfig::default_lambdas(dims) : o.lambdas;
  cfg.mu0 = o.mu0;
  cfg.mu_max = o.mu_max;
  cfg.rho = o.mu_growth;
  cfg.eps = o.eps;
  cfg.maxiter = o.maxiter;
  cfg.output_weights = o.alphas;
  return cfg;  // SnnConfig::validate runs inside pasd_b200_snn_recover (baselines.cpp:12-29)
}

SolverOptions options_from_manifest(const Manifest& m) {  // cli.cpp:222-242
  SolverOptions o;
  o.solver = m.get("solver");
  if (m.has("lambdas")) o.lambdas = m.get_doubles("lambdas");
  if (m.has("ranks")) o.ranks = m.get_indices("ranks");
  if (m.has("alphas")) o.alphas = m.get_doubles("alphas");
  o.mu0 = m.get_double("mu0");
  o.mu_max = m.get_double("mu_max");
  o.mu_growth = m.get_double("mu_growth");
  o.eps = m.get_double("eps");
  o.maxiter = (int)m.get_int("maxiter");
  return o;
}

double rse(const DenseTensor& x, const DenseTensor& t0) {  // synth.cpp:123-131
  if (x.dims() != t0.dims()) throw ArgumentError("rse: dimension mismatch");
  double ref = 0.0, err = 0.0;
  for (Index i = 0; i < x.size(); ++i) {
    ref += t0[i] * t0[i];
    err += (x[i] - t0[i]) * (x[i] - t0[i]);
  }
  ref = std::sqrt(ref);
  err = std::sqrt(err);
  if (ref == 0.0) return err == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
  return err / ref;
}

double nuclear_norm_unfold(const DenseTensor& t, Index mode) {
  double out = 0.0;
  char err[1024] = {0};
  detail::check(pasd_b200_nuclear_norm_unfold(t.data(), (int32_t)t.order(), t.dims().data(), (int32_t)mode, &out, 0,
                                              err, sizeof(err)),
                err);
  return out;
}

// ------------------------------------------------------------------ synth (cli.cpp:158-208)
int do_synth(const std::vector<std::string>& argv) {
  const Args a = parse(argv, {"--dims", "--ranks", "--rank", "--corruption", "--seed", "--mode", "--out-prefix"}, {});
  if (!a.has("--dims")) throw ArgumentError("synth needs --dims");
  if (!a.has("--out-prefix")) throw ArgumentError("synth needs --out-prefix");
  const std::vector<Index> dims = to_indices(a.str("--dims"), "--dims");
  std::vector<Index> ranks;
  if (a.has("--ranks"))
    ranks = to_indices(a.str("--ranks"), "--ranks");
  else if (a.has("--rank"))
    ranks.assign(dims.size(), (Index)to_int(a.str("--rank"), "--rank"));
  else
    throw ArgumentError("synth needs --rank or --ranks");
  const double corruption = a.has("--corruption") ? to_double(a.str("--corruption"), "--corruption") : 0.05;
  const uint64_t seed = a.has("--seed") ? (uint64_t)to_int(a.str("--seed"), "--seed") : 0;
  const std::string mode = a.str("--mode", "additive");
  if (mode != "additive" && mode != "replace255") throw ArgumentError("--mode: " + mode + " not in {additive, replace255}");
  if (ranks.size() != dims.size()) throw ArgumentError("SynthSpec: ranks and dims must have the same order");
  pasd_synth_spec sp{};
  sp.order = (int32_t)dims.size();
  sp.dims = dims.data();
  sp.ranks = ranks.data();
  sp.seed = seed;
  sp.factor_kind = 0;
  sp.corrupt_mode = mode == "replace255" ? 1 : 0;
  sp.corruption = corruption;
  sp.lo = mode == "replace255" ? 0.0 : -1.0;
  sp.hi = mode == "replace255" ? 255.0 : 1.0;
  DenseTensor truth = DenseTensor::zeros(dims), observed = DenseTensor::zeros(dims);
  int64_t count = 0;
  char err[1024] = {0};
  detail::check(pasd_b200_synth(&sp, observed.data(), 0, truth.data(), 0, nullptr, &count, err, sizeof(err)), err);
  const std::string prefix = a.str("--out-prefix");
  const fs::path tp = prefix + "_truth.tnsr", op = prefix + "_observed.tnsr";
  ensure_parent_dir(tp);
  write_tensor(truth, tp);
  write_tensor(observed, op);
  Manifest m;
  m.set_int("manifest_version", 1);
  m.set("command", "synth");
  m.set_indices("dims", dims);
  m.set_indices("ranks", ranks);
  m.set_double("corruption", corruption);
  m.set_int("seed", (long long)seed);
  m.set("corrupt_mode", mode);
  m.set("truth_out", tp.string());
  m.set("observed_out", op.string());
  m.set("truth_checksum", checksum_hex(tensor_checksum(truth)));
  m.set("observed_checksum", checksum_hex(tensor_checksum(observed)));
  m.set_int("corrupted_entries", (long long)count);
  m.save(prefix + "_synth.manifest");
  std::cout << "wrote " << tp.string() << " and " << op.string() << " (" << count << " corrupted entries)\n";
  return 0;
}

// ------------------------------------------------------------------ recover (cli.cpp:244-354)
int do_recover(const std::vector<std::string>& argv) {
  std::vector<std::string> opts = {"--input", "--truth", "--out-prefix", "--from-manifest"};
  opts.insert(opts.end(), kSolverOpts.begin(), kSolverOpts.end());
  const Args a = parse(argv, opts, {"--strict", "--no-z"});
  SolverOptions so = solver_options(a);
  std::string input = a.str("--input"), truth_path = a.str("--truth");
  if (a.has("--from-manifest")) {
    const Manifest m = Manifest::load(a.str("--from-manifest"));
    if (m.get("command") != "recover") throw ArgumentError("--from-manifest expects a recover manifest");
    so = options_from_manifest(m);
    input = m.get("input");
    if (truth_path.empty() && m.has("truth")) truth_path = m.get("truth");
  }
  if (input.empty()) throw ArgumentError("recover needs --input (or --from-manifest)");
  if (!a.has("--out-prefix")) throw ArgumentError("recover needs --out-prefix");
  if (so.solver == "rpca")
    throw ArgumentError("solver 'rpca' is not part of this build (PASD hot path and the SNN baseline only)");
  const std::string prefix = a.str("--out-prefix");
  const DenseTensor observed = read_tensor(input);
  const std::vector<Index>& dims = observed.dims();
  Manifest man;
  man.set_int("manifest_version", 1);
  man.set("command", "recover");
  man.set("solver", so.solver);
  man.set("input", input);
  man.set("input_checksum", checksum_hex(tensor_checksum(observed)));
  man.set_indices("dims", dims);
  const auto start = std::chrono::steady_clock::now();
  RecoveryResult res;
  if (so.solver == "pasd") {  // cli.cpp:272-277
    const PasdConfig cfg = build_pasd_config(so, dims);
    res = pasd_recover(observed, cfg);
    man.set_doubles("lambdas", cfg.lambdas);
    man.set_indices("ranks", cfg.ranks);
    man.set_doubles("alphas", cfg.alphas());
  } else {  // snn (cli.cpp:278-282)
    const SnnConfig cfg = build_snn_config(so, dims);
    res = snn_recover(observed, cfg);
    man.set_doubles("lambdas", cfg.lambdas);
    man.set_doubles("alphas", cfg.alphas());
  }
  const double elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  man.set_double("mu0", so.mu0);
  man.set_double("mu_max", so.mu_max);
  man.set_double("mu_growth", so.mu_growth);
  man.set_double("eps", so.eps);
  man.set_int("maxiter", so.maxiter);
  const fs::path xp = prefix + "_x.tnsr", ep = prefix + "_e.tnsr";
  ensure_parent_dir(xp);
  write_tensor(res.x, xp);
  write_tensor(res.e, ep);
  man.set("x_out", xp.string());
  man.set("e_out", ep.string());
  if (!a.flag.count("--no-z")) {
    std::string zl;
    for (size_t n = 0; n < res.z.size(); ++n) {
      const fs::path zp = prefix + "_z" + std::to_string(n + 1) + ".tnsr";
      write_tensor(res.z[n], zp);
      zl += (n ? "," : "") + zp.string();
    }
    man.set("z_out", zl);
  }
  man.set_bool("converged", res.converged);
  man.set_int("iters", res.iters);
  man.set_double("time_s", elapsed);
  man.set_doubles("final_residuals", res.final_residuals);
  man.set_double("objective", res.objective);
  if (res.certificate) {
    man.set_double("cert_epsilon_hat", res.certificate->epsilon_hat);
    man.set_double("cert_c", res.certificate->c);
    man.set_double("cert_bound", res.certificate->bound);
  }
  double rse_value = std::numeric_limits<double>::quiet_NaN();
  if (!truth_path.empty()) {
    const DenseTensor truth = read_tensor(truth_path);
    rse_value = rse(res.x, truth);
    man.set("truth", truth_path);
    man.set_double("rse", rse_value);
  }
  const fs::path mp = prefix + ".manifest";
  man.save(mp);
  std::cout << "solver = " << so.solver << ", dims =";
  for (Index d : dims) std::cout << ' ' << d;
  std::cout << "\nconverged = " << (res.converged ? "true" : "false") << " after " << res.iters << " iterations in "
            << format_double(elapsed) << " s\n";
  std::cout << "objective = " << format_double(res.objective) << "\n";
  if (!std::isnan(rse_value)) std::cout << "rse = " << format_double(rse_value) << "\n";
  if (res.certificate)
    std::cout << "certificate: epsilon_hat = " << format_double(res.certificate->epsilon_hat)
              << ", c = " << format_double(res.certificate->c) << ", bound = " << format_double(res.certificate->bound)
              << "\n";
  std::cout << "wrote " << mp.string() << "\n";
  return (a.flag.count("--strict") && !res.converged) ? 4 : 0;  // cli.cpp:351-352
}

// ------------------------------------------------------------------ certify (cli.cpp:457-553)
int do_certify(const std::vector<std::string>& argv) {
  const Args a = parse(argv, {"--manifest", "--truth"}, {});
  if (!a.has("--manifest")) throw ArgumentError("certify needs --manifest");
  const Manifest m = Manifest::load(a.str("--manifest"));
  if (m.get("command") != "recover" || m.get("solver") != "pasd")
    throw ArgumentError("certify needs a manifest written by `recover --solver pasd`");
  if (!m.has("cert_epsilon_hat")) throw ArgumentError("manifest carries no certificate (run did not converge?)");
  const DenseTensor t = read_tensor(m.get("input"));
  if (checksum_hex(tensor_checksum(t)) != m.get("input_checksum"))
    throw IoError("input tensor checksum does not match the manifest");
  const DenseTensor e = read_tensor(m.get("e_out"));
  std::vector<DenseTensor> z;
  for (const std::string& p : m.split("z_out")) z.push_back(read_tensor(p));
  const std::vector<double> lambdas = m.get_doubles("lambdas");
  const double eps = m.get_double("eps"), mu0 = m.get_double("mu0"), growth = m.get_double("mu_growth");
  const long long iters = m.get_int("iters");
  const double eps_hat = m.get_double("cert_epsilon_hat"), c_stored = m.get_double("cert_c");
  const double bound_stored = m.get_double("cert_bound"), objective = m.get_double("objective");
  if (z.size() != lambdas.size() || z.size() != t.dims().size())
    throw IoError("manifest z_out list does not cover every mode");
  bool all_ok = true;
  auto report = [&](const std::string& name, bool ok, const std::string& detail) {
    std::cout << (ok ? "[ OK ] " : "[FAIL] ") << name << ": " << detail << "\n";
    all_ok = all_ok && ok;
  };
  double worst = 0.0;  // feasibility of the stored iterate
  for (size_t n = 0; n < z.size(); ++n)
    for (Index i = 0; i < t.size(); ++i) worst = std::max(worst, std::fabs(t[i] - z[n][i] - e[i]));
  report("feasibility", worst < eps,
         "max_n |T - Z_n - E|_inf = " + format_double(worst) + " vs eps = " + format_double(eps));
  double obj = 0.0;  // ||E||_1 + sum_n lambda_n ||unfold_n(Z_n)||_* (nuclear norms on the device)
  for (Index i = 0; i < e.size(); ++i) obj += std::fabs(e[i]);
  for (size_t n = 0; n < z.size(); ++n) obj += lambdas[n] * nuclear_norm_unfold(z[n], (Index)n + 1);
  report("objective", std::fabs(obj - objective) <= 1e-6 * (1.0 + std::fabs(objective)),
         "recomputed " + format_double(obj) + " vs stored " + format_double(objective));
  const double nm = (double)t.dims().size(), total = (double)t.size();
  const double geom = growth * (1.0 + growth) / (growth - 1.0) + 0.5 / std::pow(growth, (int)iters - 1);
  double tl1 = 0.0;
  for (Index i = 0; i < t.size(); ++i) tl1 += std::fabs(t[i]);
  const double c_re = nm * total * geom / (mu0 * nm * nm) + tl1;
  report("constant_c", std::fabs(c_re - c_stored) <= 1e-12 * c_re,
         "recomputed " + format_double(c_re) + " vs stored " + format_double(c_stored));
  double lam_sum = 0.0, lam_term = 0.0;
  for (double l : lambdas) {
    lam_sum += l;
    lam_term += l * total * eps;
  }
  const double bound_re = c_re * eps_hat + lam_term;
  report("bound", std::fabs(bound_re - bound_stored) <= 1e-12 * (1.0 + bound_re),
         "recomputed " + format_double(bound_re) + " vs stored " + format_double(bound_stored));
  report("epsilon_hat", eps_hat <= 1.0 + lam_sum + 1e-9,
         format_double(eps_hat) + " <= 1 + sum(lambda) = " + format_double(1.0 + lam_sum));
  std::string tpath = a.str("--truth");
  if (tpath.empty() && m.has("truth")) tpath = m.get("truth");
  if (!tpath.empty()) {
    const DenseTensor truth = read_tensor(tpath);
    double f = 0.0;
    for (Index i = 0; i < t.size(); ++i) f += std::fabs(t[i] - truth[i]);
    for (size_t n = 0; n < lambdas.size(); ++n) f += lambdas[n] * nuclear_norm_unfold(truth, (Index)n + 1);
    report("gap_bound", objective <= f + bound_stored,
           "f* = " + format_double(objective) + " vs f_feasible + bound = " + format_double(f + bound_stored));
  }
  return all_ok ? 0 : 3;
}

int do_defaults() {  // cli.cpp:557-567
  std::cout << "mu0 = " << format_double(kDefaultMu0) << "\n";
  std::cout << "mu_max = " << format_double(kDefaultMuMax) << "\n";
  std::cout << "mu_growth = " << format_double(kDefaultMuGrowth) << "\n";
  std::cout << "eps = " << format_double(kDefaultEps) << "\n";
  std::cout << "maxiter = " << kDefaultMaxiter << "\n";
  std::cout << "lambda_rule = sqrt(max(I_n, prod_{j!=n} I_j)) / N\n";
  std::cout << "rank_bound_rule = floor(1.2 * target_rank)\n";
  std::cout << "rpca_lambda_rule = 1 / sqrt(max(rows, cols))\n";
  return 0;
}

const char* kUsage =
    "usage: tenrec_b200 <synth|recover|certify|defaults> [options]\n"
    "  synth    --dims I1,I2,.. (--rank r | --ranks r1,..) [--corruption 0.05] [--seed 0]\n"
    "           [--mode additive|replace255] --out-prefix P\n"
    "  recover  (--input T.tnsr | --from-manifest M) --out-prefix P [--truth L.tnsr] [--strict] [--no-z]\n"
    "           [--solver pasd] [--lambdas ..] [--ranks ..|--target-rank r] [--alphas ..] [--mu0 ..]\n"
    "           [--mu-max ..] [--mu-growth ..] [--eps ..] [--maxiter ..]\n"
    "  certify  --manifest M [--truth L.tnsr]\n"
    "  defaults\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage;
    return 1;
  }
  const std::string cmd = argv[1];
  const std::vector<std::string> rest(argv + 2, argv + argc);
  try {
    if (cmd == "synth") return do_synth(rest);
    if (cmd == "recover") return do_recover(rest);
    if (cmd == "certify") return do_certify(rest);
    if (cmd == "defaults") return do_defaults();
    if (cmd == "--help" || cmd == "-h") {
      std::cout << kUsage;
      return 0;
    }
    std::cerr << "error: unknown subcommand '" << cmd << "'\n" << kUsage;
    return 1;
  } catch (const ArgumentError& e) {  // cli.cpp:655-667
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const NumericalError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const StateError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const DeviceError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
}

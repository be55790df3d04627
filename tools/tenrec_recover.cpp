// tenrec_recover — minimal C++ client of the drop-in API (include/tenrec_b200/pasd.hpp):
// reads a TNSR tensor (proj/src/io.cpp:85-149 format), runs pasd_recover on the
// B200 with the reference defaults (cli.cpp:27-31, PasdConfig::default_lambdas,
// R = floor(1.2 r)), writes X and E as TNSR, prints a summary line.
//   tenrec_recover <in.tnsr> <target_rank> <out_prefix> [eps] [maxiter]
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>

#include "tenrec_b200/pasd.hpp"

using namespace tenrec_b200;

static DenseTensor read_tnsr(const char* path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError(std::string("cannot open '") + path + "' for reading");
  char magic[4];
  in.read(magic, 4);
  if (std::memcmp(magic, "TNSR", 4) != 0) throw IoError(std::string("'") + path + "': bad magic at byte offset 0 (expected \"TNSR\")");
  uint16_t hdr[2];
  in.read(reinterpret_cast<char*>(hdr), 4);
  std::vector<Index> dims(hdr[1]);
  for (auto& d : dims) {
    uint64_t v;
    in.read(reinterpret_cast<char*>(&v), 8);
    d = static_cast<Index>(v);
  }
  Index n = 1;
  for (Index d : dims) n *= d;
  std::vector<double> data(static_cast<size_t>(n));
  in.read(reinterpret_cast<char*>(data.data()), 8 * n);
  if (in.gcount() != 8 * n) throw IoError(std::string("'") + path + "': truncated payload");
  return DenseTensor::from_data(dims, std::move(data));
}

static void write_tnsr(const DenseTensor& t, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  out.write("TNSR", 4);
  uint16_t hdr[2] = {1, static_cast<uint16_t>(t.order())};
  out.write(reinterpret_cast<const char*>(hdr), 4);
  for (Index d : t.dims()) {
    uint64_t v = static_cast<uint64_t>(d);
    out.write(reinterpret_cast<const char*>(&v), 8);
  }
  out.write(reinterpret_cast<const char*>(t.data()), 8 * t.size());
}

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s <in.tnsr> <target_rank> <out_prefix> [eps] [maxiter]\n", argv[0]);
    return 1;
  }
  try {
    const DenseTensor t = read_tnsr(argv[1]);
    PasdConfig cfg;
    cfg.lambdas = PasdConfig::default_lambdas(t.dims());
    const Index r = PasdConfig::default_rank_bound(std::atoll(argv[2]));
    cfg.ranks.assign(t.dims().size(), r);
    if (argc > 4) cfg.eps = std::atof(argv[4]);
    if (argc > 5) cfg.maxiter = std::atoi(argv[5]);
    cfg.validate(t.dims());
    const RecoveryResult res = pasd_recover(t, cfg);
    write_tnsr(res.x, std::string(argv[3]) + "_x.tnsr");
    write_tnsr(res.e, std::string(argv[3]) + "_e.tnsr");
    std::printf("{\"iters\": %d, \"converged\": %s, \"objective\": %.17g, \"epsilon_hat\": %.17g}\n", res.iters,
                res.converged ? "true" : "false", res.objective,
                res.certificate ? res.certificate->epsilon_hat : -1.0);
    return 0;
  } catch (const ArgumentError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;  // cli.hpp:9-14 exit codes
  } catch (const IoError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const NumericalError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}

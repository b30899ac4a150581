// eigmod_b200: the reference CLI's update and locate subcommands
// (proj/tools/eigmod.cpp:122-161, options :262-279, exit codes :21-22 and
// :299-313) on the GPU pipeline. Same options, output files and exit codes:
//   update --eigen q.csv lambda.csv --update k.csv [--signs +1,-1] [--tol t]
//          --out prefix        -> prefix_lambda.csv, prefix_q.csv, JSON line
//   locate --eigen q.csv lambda.csv --update k.csv [--signs ...]
//          -> comma-separated location vector
// --matrix (Matrix Market input decomposed by the CPU Jacobi baseline) is out
// of scope and is rejected as a usage error.
#include <charconv>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

#include "eigmod/eigvec.hpp"
#include "eigmod/io.hpp"
#include "eigmod/locate.hpp"
#include "eigmod/secular.hpp"

namespace {

constexpr int kExitUsage = 2;
constexpr int kExitNumerical = 3;

struct UpdateArgs {
  std::string matrix_path;
  std::vector<std::string> eigen_paths;
  std::string update_path;
  std::string signs;
  double tol = 0.0;
  std::string out_prefix;
};

std::string num(double v) {
  char b[40];
  auto r = std::to_chars(b, b + 40, v);
  return std::string(b, r.ptr);
}

eigmod::SpectralDecomposition load_decomposition(const UpdateArgs& a) {
  if (!a.matrix_path.empty())
    throw std::invalid_argument(
        "--matrix needs the CPU Jacobi decomposition, which this build does not ship; "
        "pass --eigen q.csv lambda.csv");
  if (a.eigen_paths.size() != 2)
    throw eigmod::FormatError("either --matrix or --eigen <q.csv> <lambda.csv> is required");
  eigmod::SpectralDecomposition d;
  d.q = eigmod::read_csv_matrix(a.eigen_paths[0]).values;
  const eigmod::Matrix lam = eigmod::read_csv_matrix(a.eigen_paths[1]).values;
  if (lam.cols() == 1) {
    d.lambda.resize(lam.rows());
    for (std::size_t i = 0; i < lam.rows(); ++i) d.lambda[i] = lam(i, 0);
  } else if (lam.rows() == 1) {
    d.lambda.resize(lam.cols());
    for (std::size_t j = 0; j < lam.cols(); ++j) d.lambda[j] = lam(0, j);
  } else {
    throw eigmod::FormatError(a.eigen_paths[1] + ": eigenvalues must be a single column or row");
  }
  eigmod::validate_decomposition(d);
  return d;
}

eigmod::LowRankUpdate load_update(const UpdateArgs& a, std::size_t n) {
  if (a.update_path.empty()) throw eigmod::FormatError("--update is required");
  const eigmod::CsvMatrix k = eigmod::read_csv_matrix(a.update_path);
  eigmod::LowRankUpdate u;
  u.kmat = k.values;
  if (u.kmat.rows() != n)
    throw eigmod::FormatError(a.update_path + ": row count does not match the matrix size");
  if (!a.signs.empty()) u.signs = eigmod::parse_signs(a.signs);
  else if (k.signs) u.signs = *k.signs;
  else u.signs.assign(u.kmat.cols(), 1);
  if (u.signs.size() != u.kmat.cols())
    throw eigmod::FormatError("sign count does not match the update rank");
  return u;
}

int cmd_update(const UpdateArgs& a) {
  const eigmod::SpectralDecomposition d = load_decomposition(a);
  const eigmod::LowRankUpdate u = load_update(a, d.size());
  const double tol = a.tol > 0.0 ? a.tol : eigmod::default_tolerance(d.lambda, u);
  const eigmod::UpdateResult res = eigmod::update_decomposition(d, u, tol);
  eigmod::Matrix lam(res.decomposition.lambda.size(), 1);
  for (std::size_t i = 0; i < lam.rows(); ++i) lam(i, 0) = res.decomposition.lambda[i];
  eigmod::write_csv_matrix(a.out_prefix + "_lambda.csv", lam);
  eigmod::write_csv_matrix(a.out_prefix + "_q.csv", res.decomposition.q);
  // nlohmann::json object order (keys sorted), as the reference prints it
  std::cout << "{\"k\":" << u.rank() << ",\"n\":" << d.size()
            << ",\"ortho_err\":" << num(res.ortho_err)
            << ",\"residual_fro\":" << num(res.residual_fro)
            << ",\"wall_time\":" << num(res.wall_time) << "}\n";
  return 0;
}

int cmd_locate(const UpdateArgs& a) {
  const eigmod::SpectralDecomposition d = load_decomposition(a);
  const eigmod::LowRankUpdate u = load_update(a, d.size());
  const eigmod::LocationVector loc = eigmod::locate_update(d, u);
  for (std::size_t i = 0; i < loc.counts.size(); ++i)
    std::cout << (i ? "," : "") << loc.counts[i];
  std::cout << "\n";
  return 0;
}

int usage(const char* msg) {
  std::cerr << msg << "\n"
            << "usage: eigmod_b200 [--parallel] update|locate --eigen Q.csv LAMBDA.csv "
               "--update K.csv [--signs S] [--tol T] [--out PREFIX]\n";
  return kExitUsage;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  std::string sub;
  UpdateArgs a;
  for (std::size_t i = 0; i < args.size(); ++i) {
    const std::string& t = args[i];
    auto value = [&](const char* opt) -> std::string {
      if (i + 1 >= args.size()) throw std::invalid_argument(std::string(opt) + " needs a value");
      return args[++i];
    };
    try {
      if (t == "--parallel") continue;  // the OpenMP toggle has no GPU meaning
      if (t == "-h" || t == "--help") return usage("low-rank spectral updates (B200)") == 0;
      if (sub.empty() && (t == "update" || t == "locate")) {
        sub = t;
      } else if (sub.empty()) {
        return usage(("unknown subcommand '" + t + "'").c_str());
      } else if (t == "--matrix") {
        a.matrix_path = value("--matrix");
      } else if (t == "--eigen") {
        a.eigen_paths.push_back(value("--eigen"));
        a.eigen_paths.push_back(value("--eigen"));
      } else if (t == "--update") {
        a.update_path = value("--update");
      } else if (t == "--signs") {
        a.signs = value("--signs");
      } else if (t == "--tol" && sub == "update") {
        a.tol = std::stod(value("--tol"));
      } else if (t == "--out" && sub == "update") {
        a.out_prefix = value("--out");
      } else {
        return usage(("unknown option '" + t + "'").c_str());
      }
    } catch (const std::exception& e) {
      return usage(e.what());
    }
  }
  if (sub.empty()) return usage("a subcommand is required");
  if (a.update_path.empty()) return usage("--update is required");
  if (sub == "update" && a.out_prefix.empty()) return usage("--out is required");
  try {
    return sub == "update" ? cmd_update(a) : cmd_locate(a);
  } catch (const eigmod::NumericalError& e) {
    std::cerr << "numerical failure at stage '" << e.stage() << "': " << e.what() << "\n";
    return kExitNumerical;
  } catch (const eigmod::FormatError& e) {
    std::cerr << "input error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::invalid_argument& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitNumerical;
  }
}

// rank-bench — the SPEC cli `rank-bench` subcommand on the B200 path.
//
//   rank-bench --d D --interaction far|surface:K --kernel NAME[,NAME...] --N n1[,n2...]
//              [--epsilon 1e-12] [--grid uniform|interior|closed] [--seed S] [--devices 0[,1..]]
//              [--out file.csv] [--fit 1]
//
// --fit 1: after the CSV, SPEC fit_growth of every kernel's rank(N) series with
// at least 4 distinct N, one "# fit ..." line per kernel on stderr.
//
// NAME is a catalog kernel (kernel.hpp:112-129) or one of the paper's complex columns
// "helmholtz3d" (F3 = e^{ir}/r) and "hankel_h12" (F4 = H_2^(1)(r)), ranked as K_re + i·K_im.
//
// Prints the CSV of SPEC.md:613 (plus certification columns).  Exit codes (SPEC.md:666,
// run_rank_bench): 0 success, 2 some problems skipped by a guard (ENOMEM/ECAP), 1 error,
// 64 usage error (missing / malformed flag).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "hb200.hpp"

namespace {

int usage(const char* msg) {
  std::fprintf(stderr,
               "rank-bench: %s\nusage: rank-bench --d D --interaction far|surface:K --kernel NAME[,..] "
               "--N n1[,..] [--epsilon E] [--grid uniform|interior|closed] [--seed S] "
               "[--devices 0,..] [--out FILE] [--fit 1]\n",
               msg);
  return 64;
}

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ','))
    if (!tok.empty()) out.push_back(tok);
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> a;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0 || i + 1 >= argc) return usage(("bad argument " + k).c_str());
    a[k.substr(2)] = argv[++i];
  }
  for (const char* req : {"d", "interaction", "kernel", "N"})
    if (!a.count(req)) return usage((std::string("missing --") + req).c_str());
  try {
    const int d = std::stoi(a["d"]);
    const auto inter = hb200::InteractionClass::parse(a["interaction"]);
    std::vector<hb200::KernelSpec> kernels;
    std::vector<std::pair<hb200::KernelSpec, hb200::KernelSpec>> complex_kernels;
    for (const auto& k : split(a["kernel"])) {
      if (k == "helmholtz3d")  // F3
        complex_kernels.push_back({hb200::kernel_from_string("helmholtz3d_re"),
                                   hb200::kernel_from_string("helmholtz3d_im")});
      else if (k == "hankel_h12")  // F4
        complex_kernels.push_back({hb200::kernel_from_string("hankel_h12_re"),
                                   hb200::kernel_from_string("hankel_h12_im")});
      else
        kernels.push_back(hb200::kernel_from_string(k));
    }
    std::vector<int64_t> ns;
    for (const auto& n : split(a["N"])) ns.push_back(std::stoll(n));
    const double eps = a.count("epsilon") ? std::stod(a["epsilon"]) : 1e-12;
    hb200::PointMode mode = hb200::PointMode::Uniform;
    if (a.count("grid")) {
      if (a["grid"] == "interior") mode = hb200::PointMode::GridInterior;
      else if (a["grid"] == "closed") mode = hb200::PointMode::GridClosed;
      else if (a["grid"] != "uniform") return usage("--grid must be uniform|interior|closed");
    }
    const uint64_t seed = a.count("seed") ? std::stoull(a["seed"]) : 0;
    std::vector<int> devs = {0};
    if (a.count("devices")) {
      devs.clear();
      for (const auto& s : split(a["devices"])) devs.push_back(std::stoi(s));
    }
    std::vector<hb_status> st;
    auto recs = kernels.empty() ? std::vector<hb200::RankRecord>{}
                                : hb200::rank_table(kernels, inter, d, ns, eps, devs, mode, seed, &st);
    if (!complex_kernels.empty()) {  // complex columns: one problem at a time on the first device
      hb200::Device dev(devs.front());
      for (const auto& kk : complex_kernels)
        for (const int64_t n : ns) {
          const uint64_t ps = mode == hb200::PointMode::Uniform ? hb200::problem_seed(seed, d, inter, n) : seed;
          const auto g = hb200::pair_geometry(d, inter, n, mode, ps);
          try {
            recs.push_back(hb200::epsilon_rank_complex(dev, kk.first, kk.second, g, {eps}).front());
            st.push_back(HB_OK);
          } catch (const std::length_error&) {
            hb200::RankRecord r;
            r.kernel = hb200::kernel_name(kk.first) + "+i*" + hb200::kernel_name(kk.second);
            r.N = n;
            recs.push_back(r);
            st.push_back(HB_ECAP);
          }
        }
    }
    std::ofstream f;
    std::ostream* os = &std::cout;
    if (a.count("out")) {
      f.open(a["out"]);
      os = &f;
    }
    hb200::write_csv_header(*os);
    int rc = 0;
    for (size_t i = 0; i < recs.size(); ++i) {
      if (st[i] == HB_OK) {
        hb200::write_csv_row(*os, recs[i]);
      } else if (st[i] == HB_ENOMEM || st[i] == HB_ECAP) {
        std::fprintf(stderr, "skipped %s N=%lld: %s\n", recs[i].kernel.c_str(), (long long)recs[i].N,
                     hb_status_string(st[i]));
        if (rc == 0) rc = 2;
      } else {
        std::fprintf(stderr, "error %s N=%lld: %s\n", recs[i].kernel.c_str(), (long long)recs[i].N,
                     hb_status_string(st[i]));
        rc = 1;
      }
    }
    if (a.count("fit") && a["fit"] != "0") {
      std::map<std::string, std::vector<hb200::RankRecord>> by;
      for (size_t i = 0; i < recs.size(); ++i)
        if (st[i] == HB_OK) by[recs[i].kernel].push_back(recs[i]);
      for (const auto& [name, series] : by) {
        try {
          const auto g = hb200::fit_growth(series);
          std::fprintf(stderr, "# fit %s: best %s, constant %.3f, log %.3f + %.3f ln N, power %.4g N^%.4f, "
                       "rss %.4g/%.4g/%.4g, max/min %.3f\n", name.c_str(), g.best.c_str(), g.constant,
                       g.log_a, g.log_b, g.pow_a, g.pow_c, g.rss[0], g.rss[1], g.rss[2], g.max_min_ratio);
        } catch (const std::invalid_argument& e) {
          std::fprintf(stderr, "# fit %s: refused (%s)\n", name.c_str(), e.what());
        }
      }
    }
    hb_sweep_release();
    return rc;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "rank-bench: %s\n", e.what());
    return 64;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rank-bench: %s\n", e.what());
    return 1;
  }
}

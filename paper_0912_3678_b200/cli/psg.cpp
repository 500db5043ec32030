// psg -- command-line surface of the solver (the reference's planned `parsol`
// tool, SPEC.md "MODULE cli"; its tools/parsol.cpp is a stub): generation,
// solving, verification, partition plans and benchmarking on the B200, with
// the reference's STRUCTMAT / VEC files (include/parsol/io.hpp).
//
//   psg generate --kind K --n N [--m M --s S --r R] --seed X --dominance D -o A.mat [--rhs F.vec]
//   psg generate --config C --size Z --seed X -o A.mat [--rhs F.vec]     (BASELINE configs)
//   psg solve    -m A.mat -f F.vec|ones --p P [--strategy lu] [-o X.vec] [--exact]
//   psg verify   -m A.mat -f F.vec|ones --p P [--strategy lu] [--tol T]
//   psg plan     -m A.mat --p P
//   psg bench    --config C --size Z --p P [--reps R] [--seed X]
//   psg ode      --problem heat|decay --m M [--lambda L] --p P --N N [--method ie|trap] [--T T] [-o Y.traj]
//   psg parareal --problem heat|decay --m M --p P --N N [--method ie|trap] [--coarse ie|trap|expm]
//                [--coarse-steps C] [--tol T] [--max-iter K] [-o H.csv]
//
// Exit codes: 0 ok, 1 usage / parse / I/O error, 2 numeric failure; errors
// are reported on stderr as `ERROR <code> <detail>`.  Benchmark output is CSV
// `phase,n,p,workers,median_seconds,op_count` (medians of --reps runs, device
// timing; workers = 1 GPU).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "parsol/errors.hpp"
#include "parsol/io.hpp"
#include "parsol/odeparallel.hpp"
#include "parsol/parareal.hpp"
#include "parsol/parfact.hpp"
#include "parsol/partition.hpp"
#include "parsol/seqref.hpp"
#include "psg.h"

using namespace parsol;

namespace {

struct Args {
  std::string cmd;
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string str(const std::string& k, const std::string& def = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? def : it->second;
  }
  long num(const std::string& k, long def) const { return has(k) ? std::stol(str(k)) : def; }
  double real(const std::string& k, double def) const { return has(k) ? std::stod(str(k)) : def; }
  std::string need(const std::string& k) const {
    if (!has(k)) fail(Errc::InvalidParameter, "missing --" + k);
    return str(k);
  }
};

Args parse_args(int argc, char** argv) {
  if (argc < 2) fail(Errc::InvalidParameter, "usage: psg <generate|solve|verify|plan|bench|ode|parareal> [options]");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k == "-o") k = "--out";
    if (k == "-m") k = "--matrix";
    if (k == "-f") k = "--rhs-in";
    if (k.rfind("--", 0) != 0) fail(Errc::InvalidParameter, "unexpected argument '" + k + "'");
    k = k.substr(2);
    if (k == "exact") {
      a.kv[k] = "1";
      continue;
    }
    if (i + 1 >= argc) fail(Errc::InvalidParameter, "--" + k + " needs a value");
    a.kv[k] = argv[++i];
  }
  return a;
}

void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) fail(Errc::Cuda, cudaGetErrorString(e));
}
void psg_check(int rc, const char* err) {
  if (rc) fail(Errc(rc - 1), err);
}

// BASELINE config instance, generated on the device and copied to the host
StructuredMatrix config_matrix(int cfg, int size, std::uint64_t seed, Vector* f) {
  int kind, n, m, s, r, cr, cc;
  size_t len;
  if (psg_config_shape(cfg, size, &kind, &n, &m, &s, &r, &len, &cr, &cc))
    fail(Errc::InvalidParameter, "unknown config " + std::to_string(cfg));
  double *dd = nullptr, *dc = nullptr, *df = nullptr;
  cuda_check(cudaMalloc(&dd, sizeof(double) * len));
  cuda_check(cudaMalloc(&dc, sizeof(double) * std::max(1, cr * cc)));
  cuda_check(cudaMalloc(&df, sizeof(double) * n));
  char err[512] = {0};
  psg_check(psg_generate_config(cfg, size, seed, dd, dc, df, nullptr, err, sizeof err), err);
  std::vector<double> data(len), corner(std::size_t(cr) * cc);
  f->resize(n);
  cuda_check(cudaMemcpy(data.data(), dd, sizeof(double) * len, cudaMemcpyDeviceToHost));
  if (!corner.empty()) cuda_check(cudaMemcpy(corner.data(), dc, sizeof(double) * corner.size(), cudaMemcpyDeviceToHost));
  cuda_check(cudaMemcpy(f->data(), df, sizeof(double) * n, cudaMemcpyDeviceToHost));
  cudaFree(dd);
  cudaFree(dc);
  cudaFree(df);
  return make(Kind(kind), n, m, s, r, std::move(data), std::move(corner), cr, cc);
}

Vector rhs_of(const Args& a, int n) {
  const std::string src = a.need("rhs-in");
  if (src == "ones") return Vector(n, 1.0);
  Vector f = parse_vector(read_file(src));
  if ((int)f.size() != n) fail(Errc::DimensionMismatch, "rhs length " + std::to_string(f.size()) + " != n");
  return f;
}

int cmd_generate(const Args& a) {
  StructuredMatrix A;
  Vector f;
  std::vector<std::string> comments;
  const std::uint64_t seed = (std::uint64_t)a.num("seed", 1);
  if (a.has("config")) {
    const int cfg = (int)a.num("config", 1), size = (int)std::stol(a.need("size"));
    A = config_matrix(cfg, size, seed, &f);
    comments.push_back("generator BASELINE config " + std::to_string(cfg) + " size " + std::to_string(size) +
                       " splitmix64 seed " + std::to_string(seed));
  } else {
    const Kind kind = kind_from_name(a.need("kind"));
    const int n = (int)std::stol(a.need("n"));
    const double dom = a.real("dominance", 2.0);
    A = generate_random(kind, n, (int)a.num("m", 1), (int)a.num("s", 1), (int)a.num("r", 1), seed, dom);
    comments.push_back("generator generate_random splitmix64 seed " + std::to_string(seed) + " dominance " +
                       format_hex(dom));
    f.assign(n, 1.0);
  }
  write_file(a.need("out"), write_matrix(A, comments));
  if (a.has("rhs")) write_file(a.str("rhs"), write_vector(f, comments));
  std::printf("wrote %s: %s n=%d m=%d s=%d r=%d\n", a.str("out").c_str(), kind_name(A.kind), A.n, A.m, A.s, A.r);
  return 0;
}

int cmd_solve(const Args& a, bool verify) {
  const StructuredMatrix A = parse_matrix(read_file(a.need("matrix")));
  const Vector f = rhs_of(a, A.n);
  const int p = (int)std::stol(a.need("p"));
  const Strategy st = strategy_from_name(a.str("strategy", "lu"));
  const auto t0 = std::chrono::steady_clock::now();
  ParallelFactorization F = parallel_factor(A, p, st);
  if (a.has("exact")) psg_set_option(F.device.get(), PSG_OPT_SPECULATIVE, 0.0);
  SolveStats stats;
  const Vector x = solve(F, f, &stats);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const double res = residual(A, x, f);
  std::printf("residual %s (%.3e)\n", format_hex(res).c_str(), res);
  std::printf("n %d p %d strategy %s q %d seconds %.6f certificate %.3e fallbacks %d\n", A.n, p, strategy_name(st),
              F.reduced.q, secs, stats.certificate, stats.fallbacks);
  if (a.has("out")) write_file(a.str("out"), write_vector(x));
  if (!verify) return 0;
  // dense oracle (partial-pivot LU of the assembled matrix) where it fits
  const double tol = a.real("tol", 1e-10);
  if (A.n > 4096) {
    std::printf("dense oracle skipped (n > 4096); residual check only\n");
    return res <= tol ? 0 : 2;
  }
  const Vector xd = lu_solve(to_dense(A, 4096), f);
  double num = 0, den = 0;
  for (int i = 0; i < A.n; ++i) {
    num = std::max(num, std::fabs(x[i] - xd[i]));
    den = std::max(den, std::fabs(xd[i]));
  }
  const double err = den > 0 ? num / den : num;
  std::printf("max relative error %s (%.3e) tol %.1e\n", format_hex(err).c_str(), err, tol);
  return err <= tol ? 0 : 2;
}

int cmd_plan(const Args& a) {
  const StructuredMatrix A = parse_matrix(read_file(a.need("matrix")));
  std::printf("%s\n", describe(plan_partition(A, (int)std::stol(a.need("p")))).c_str());
  return 0;
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0.0 : v[v.size() / 2];
}

int cmd_bench(const Args& a) {
  const int cfg = (int)a.num("config", 1), size = (int)std::stol(a.need("size")), p = (int)std::stol(a.need("p"));
  const int reps = (int)a.num("reps", 5);
  const std::uint64_t seed = (std::uint64_t)a.num("seed", cfg + 1);
  int kind, n, m, s, r, cr, cc;
  size_t len;
  if (psg_config_shape(cfg, size, &kind, &n, &m, &s, &r, &len, &cr, &cc))
    fail(Errc::InvalidParameter, "unknown config " + std::to_string(cfg));
  double *dd = nullptr, *dc = nullptr, *df = nullptr, *dx = nullptr;
  cuda_check(cudaMalloc(&dd, sizeof(double) * len));
  cuda_check(cudaMalloc(&dc, sizeof(double) * std::max(1, cr * cc)));
  cuda_check(cudaMalloc(&df, sizeof(double) * n));
  cuda_check(cudaMalloc(&dx, sizeof(double) * n));
  char err[512] = {0};
  psg_check(psg_generate_config(cfg, size, seed, dd, dc, df, nullptr, err, sizeof err), err);
  const psg_desc d{kind, n, m, s, r, dd, len, cr ? dc : nullptr, cr, cc, 1};
  std::vector<double> tf, t1, t2, t3, tt;
  long long ops = 0;
  for (int i = 0; i < reps + 1; ++i) {  // first run: warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    psg_handle* h = nullptr;
    psg_check(psg_factor(&d, p, PSG_LU, 1e-8, nullptr, &h, err, sizeof err), err);
    psg_stats st{};
    const int rc = psg_solve(h, df, dx, 1, nullptr, &st, err, sizeof err);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    psg_release(h);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    psg_check(rc, err);
    if (i == 0) continue;
    tf.push_back(st.factor_seconds);
    t1.push_back(st.phase1_seconds);
    t2.push_back(st.phase2_seconds);
    t3.push_back(st.phase3_seconds);
    tt.push_back(ms * 1e-3);
    ops = st.reduced_ops;
  }
  std::printf("phase,n,p,workers,median_seconds,op_count\n");
  std::printf("factor,%d,%d,1,%.9f,0\n", n, p, median(tf));
  std::printf("phase1,%d,%d,1,%.9f,0\n", n, p, median(t1));
  std::printf("phase2,%d,%d,1,%.9f,%lld\n", n, p, median(t2), ops);
  std::printf("phase3,%d,%d,1,%.9f,0\n", n, p, median(t3));
  std::printf("total,%d,%d,1,%.9f,%lld\n", n, p, median(tt), ops);
  cudaFree(dd);
  cudaFree(dc);
  cudaFree(df);
  cudaFree(dx);
  return 0;
}

// the bundled problems (reference parareal.hpp: heat_problem, decay_problem)
IVProblem problem_of(const Args& a) {
  const std::string pr = a.str("problem", "heat");
  const double t0 = a.real("t0", 0.0);
  if (pr == "heat") return heat_problem((int)a.num("m", 32), t0, a.real("T", 0.1));
  if (pr == "decay") return decay_problem(a.real("lambda", -1.0), t0, a.real("T", 1.0));
  fail(Errc::InvalidParameter, "unknown problem '" + pr + "' (heat, decay)");
}

int cmd_ode(const Args& a) {
  const IVProblem prob = problem_of(a);
  const int p = (int)std::stol(a.need("p")), N = (int)std::stol(a.need("N"));
  const OdeMethod meth = method_from_name(a.str("method", "ie"));
  const TimeGrid grid = coarse_mesh(prob.t0, prob.T, p, N);
  SolveStats st;
  const auto t0 = std::chrono::steady_clock::now();
  const Trajectory tr = solve_ivp_parallel(prob, grid, meth, &st);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (a.has("out")) write_file(a.str("out"), write_trajectory(tr.flat, tr.m, tr.p, tr.N));
  const Vector e = tr.endpoint();
  std::printf("m %d p %d N %d method %s seconds %.6f certificate %.3e\n", tr.m, p, N, method_name(meth), secs,
              st.certificate);
  std::printf("endpoint[0] %s (%.15e)\n", format_hex(e[0]).c_str(), e[0]);
  return 0;
}

int cmd_parareal(const Args& a) {
  const IVProblem prob = problem_of(a);
  const int p = (int)std::stol(a.need("p")), N = (int)std::stol(a.need("N"));
  Propagator fine;
  fine.kind = PropagatorKind::FineDiscrete;
  fine.method = method_from_name(a.str("method", "ie"));
  fine.steps = N;
  Propagator coarse;
  const std::string cs = a.str("coarse", "ie");
  coarse.kind = cs == "expm" ? PropagatorKind::MatrixExponential : PropagatorKind::CoarseDiscrete;
  coarse.method = cs == "expm" ? OdeMethod::ImplicitEuler : method_from_name(cs);
  coarse.steps = (int)a.num("coarse-steps", 1);
  const TimeGrid grid = coarse_mesh(prob.t0, prob.T, p, N);
  const auto t0 = std::chrono::steady_clock::now();
  const PararealResult r = parareal_solve(prob, grid, fine, coarse, a.real("tol", 1e-8), (int)a.num("max-iter", -1));
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::string csv = "iter,update_norm\n";
  for (std::size_t k = 0; k < r.history.size(); ++k) csv += std::to_string(k + 1) + "," + format_hex(r.history[k]) + "\n";
  if (a.has("out")) write_file(a.str("out"), csv);
  else std::fputs(csv.c_str(), stdout);
  std::printf("iterations %d converged %d seconds %.6f\n", r.iterations, r.converged ? 1 : 0, secs);
  if (!r.converged) fail(Errc::NotConverged, "no convergence in " + std::to_string(r.iterations) + " iterations");
  return 0;
}

bool numeric(Errc c) {
  switch (c) {
    case Errc::ZeroPivot:
    case Errc::SingularBlock:
    case Errc::SingularFactor:
    case Errc::SingularReducedSystem:
    case Errc::SingularWindow:
    case Errc::NotConverged:
    case Errc::ExpmFailure: return true;
    default: return false;
  }
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse_args(argc, argv);
    if (a.cmd == "generate") return cmd_generate(a);
    if (a.cmd == "solve") return cmd_solve(a, false);
    if (a.cmd == "verify") return cmd_solve(a, true);
    if (a.cmd == "plan") return cmd_plan(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "ode") return cmd_ode(a);
    if (a.cmd == "parareal") return cmd_parareal(a);
    fail(Errc::InvalidParameter, "unknown command '" + a.cmd + "'");
  } catch (const Error& e) {
    std::fprintf(stderr, "ERROR %s %s\n", errc_name(e.code()), e.detail().c_str());
    return numeric(e.code()) ? 2 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ERROR InvalidParameter %s\n", e.what());
    return 1;
  }
}

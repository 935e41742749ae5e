// cmtf_b200 -- command-line front end of the B200 path, with the reference
// CLI's train / eval subcommands (tools/cmtf_main.cpp:113-239 of the
// reference): same options, outputs (model.txt, log.csv, test.tns,
// manifest.json), printed lines and exit codes (0 ok, 2 DivergenceError,
// 1 anything else, errors as "error: <message>" on stderr).  Built on the C
// ABI only (include/cmtf_b200.h): text parsing and writing on all host
// threads, validation, training and evaluation on the device.
//
//   cmtf_b200 train --tensor T.tns --rank 10,10,10 [--split 0.1 | --test X.tns]
//                   [--couple MODE:PATH:LAMBDA ...] [--kernel naive|opt] [--cp]
//                   [--nonneg] [--eta 1e-3] [--mu 0.1] [--lreg 0.1] [--workers 1]
//                   [--epochs 100] [--tol 1e-4] [--seed 0] [--out DIR]
//   cmtf_b200 eval --model M.txt --test X.tns [--couple MODE:PATH:LAMBDA ...] [--json]
#include <sys/stat.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cmtf_b200.h"

namespace {

constexpr const char* kVersion = "0.1.0";

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void check(int rc, const cmtf_gpu_ctx* ctx = nullptr) {
  if (rc != CMTF_OK) throw Failure(rc, ctx ? cmtf_gpu_ctx_error(ctx) : cmtf_gpu_last_error());
}
[[noreturn]] void invalid(const std::string& m) { throw Failure(CMTF_EVALIDATION, m); }

// ---- data held on the host (the reference's SparseTensor / CoupledMatrix)
struct Coo {
  std::vector<uint32_t> dims, idx;
  std::vector<double> vals;
  bool header = false;
  uint64_t nnz() const { return vals.size(); }
  int order() const { return (int)dims.size(); }
};
Coo parse(const std::string& path, int expected_order) {
  cmtf_coo* c = nullptr;
  check(cmtf_coo_parse(path.c_str(), expected_order, 0, &c));
  std::unique_ptr<cmtf_coo, void (*)(cmtf_coo*)> own(c, cmtf_coo_free);
  Coo out;
  const int order = cmtf_coo_order(c);
  const uint64_t n = cmtf_coo_nnz(c);
  out.dims.assign(cmtf_coo_dims(c), cmtf_coo_dims(c) + order);
  out.idx.assign(cmtf_coo_indices(c), cmtf_coo_indices(c) + n * order);
  out.vals.assign(cmtf_coo_values(c), cmtf_coo_values(c) + n);
  out.header = cmtf_coo_has_header(c);
  return out;
}
int device() {
  const char* v = std::getenv("CMTF_DEVICE");
  return v ? std::atoi(v) : 0;
}
// load_tensor (src/sparse_data.cpp:247-254): parse + the constructor's checks
Coo load_tensor(const std::string& path) {
  Coo t = parse(path, 0);
  if (t.order() < 2) throw Failure(CMTF_EPARSE, "'" + path + "': tensor order must be at least 2");
  check(cmtf_gpu_check_entries(device(), t.order(), t.dims.data(), t.idx.data(), t.vals.data(),
                               t.nnz(), 0));
  return t;
}
struct Couple {
  int mode = 0;  // 1-based
  std::string path;
  double lambda = 10.0;
};
struct Matrix {
  int mode0;
  uint32_t rows, cols;
  std::vector<uint32_t> idx;
  std::vector<double> vals;
  double weight;
};
// load_matrix (src/sparse_data.cpp:256-277)
Matrix load_matrix(const Couple& c, const Coo& tensor) {
  if (c.mode < 1 || c.mode > tensor.order())
    invalid("coupled mode " + std::to_string(c.mode) + " out of range 1.." +
            std::to_string(tensor.order()));
  if (!(c.lambda > 0)) invalid("lambda_m must be positive");
  Coo f = parse(c.path, 2);
  const uint32_t rows = tensor.dims[c.mode - 1];
  if (f.header && f.dims[0] != rows)
    invalid("'" + c.path + "': matrix has " + std::to_string(f.dims[0]) + " rows but mode " +
            std::to_string(c.mode) + " has size " + std::to_string(rows));
  if (f.dims[0] > rows)
    invalid("'" + c.path + "': matrix row index exceeds size of mode " + std::to_string(c.mode));
  const uint32_t md[2] = {rows, f.dims[1]};
  check(cmtf_gpu_check_entries(device(), 2, md, f.idx.data(), f.vals.data(), f.nnz(), 1));
  return Matrix{c.mode - 1, rows, f.dims[1], std::move(f.idx), std::move(f.vals), c.lambda};
}

// MODE:PATH:LAMBDA, the path may contain ':' (cmtf_main.cpp:36-56)
Couple parse_couple(const std::string& arg) {
  const auto first = arg.find(':'), last = arg.rfind(':');
  if (first == std::string::npos || first == last)
    invalid("--couple expects MODE:PATH:LAMBDA, got '" + arg + "'");
  Couple c;
  try {
    c.mode = std::stoi(arg.substr(0, first));
    c.lambda = std::stod(arg.substr(last + 1));
  } catch (const std::exception&) {
    invalid("--couple expects MODE:PATH:LAMBDA, got '" + arg + "'");
  }
  c.path = arg.substr(first + 1, last - first - 1);
  if (c.path.empty()) invalid("--couple has an empty path in '" + arg + "'");
  return c;
}
std::vector<uint32_t> parse_u32_list(const std::string& arg, const char* what) {
  std::vector<uint32_t> out;
  std::string tok;
  std::istringstream ss(arg);
  while (std::getline(ss, tok, ',')) {
    try {
      const long v = std::stol(tok);
      if (v < 1) throw std::out_of_range(tok);
      out.push_back((uint32_t)v);
    } catch (const std::exception&) {
      invalid(std::string(what) + " expects a comma-separated list of positive integers, got '" +
              arg + "'");
    }
  }
  if (out.empty()) invalid(std::string(what) + " must not be empty");
  return out;
}

// ---- a little JSON writer (manifest.json; sorted keys, 2-space indent)
struct Json {
  enum Kind { Str, Num, Int, Bool, Arr, Obj, Null } kind = Null;
  std::string s;
  double d = 0;
  long long i = 0;
  bool b = false;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
  static Json str(std::string v) { Json j; j.kind = Str; j.s = std::move(v); return j; }
  static Json num(double v) { Json j; j.kind = Num; j.d = v; return j; }
  static Json integer(long long v) { Json j; j.kind = Int; j.i = v; return j; }
  static Json boolean(bool v) { Json j; j.kind = Bool; j.b = v; return j; }
  static Json array() { Json j; j.kind = Arr; return j; }
  static Json object() { Json j; j.kind = Obj; return j; }
  Json& operator[](const std::string& k) {
    kind = Obj;
    return obj[k];
  }
  void dump(std::string& o, int ind) const {
    auto pad = [&](int n) { o.append(n, ' '); };
    switch (kind) {
      case Null: o += "null"; break;
      case Bool: o += b ? "true" : "false"; break;
      case Int: o += std::to_string(i); break;
      case Num: {
        char buf[40];
        std::snprintf(buf, sizeof buf, "%.17g", d);
        for (int p = 1; p <= 17; ++p) {  // shortest round-tripping form
          char t[40];
          std::snprintf(t, sizeof t, "%.*g", p, d);
          if (std::strtod(t, nullptr) == d) {
            std::snprintf(buf, sizeof buf, "%s", t);
            break;
          }
        }
        o += buf;
        break;
      }
      case Str: {
        o += '"';
        for (char c : s) {
          if (c == '"' || c == '\\') o += '\\';
          o += c;
        }
        o += '"';
        break;
      }
      case Arr:
        if (arr.empty()) { o += "[]"; break; }
        o += "[\n";
        for (size_t k = 0; k < arr.size(); ++k) {
          pad(ind + 2);
          arr[k].dump(o, ind + 2);
          o += k + 1 < arr.size() ? ",\n" : "\n";
        }
        pad(ind);
        o += "]";
        break;
      case Obj: {
        if (obj.empty()) { o += "{}"; break; }
        o += "{\n";
        size_t k = 0;
        for (const auto& [key, v] : obj) {
          pad(ind + 2);
          o += "\"" + key + "\": ";
          v.dump(o, ind + 2);
          o += ++k < obj.size() ? ",\n" : "\n";
        }
        pad(ind);
        o += "}";
        break;
      }
    }
  }
};
void write_text(const std::string& path, const std::string& text) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw Failure(CMTF_EPARSE, "cannot write '" + path + "'");
  const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  if (std::fclose(f) != 0 || !ok) throw Failure(CMTF_EPARSE, "write failed for '" + path + "'");
}
void make_dirs(const std::string& dir) {
  std::string cur;
  std::istringstream ss(dir);
  std::string part;
  if (!dir.empty() && dir[0] == '/') cur = "/";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) continue;
    cur += part + "/";
    mkdir(cur.c_str(), 0777);
  }
}
Json argv_json(int argc, char** argv) {
  Json a = Json::array();
  for (int k = 0; k < argc; ++k) a.arr.push_back(Json::str(argv[k]));
  return a;
}

// ---- options
struct Opts {
  std::map<std::string, std::string> val;
  std::vector<std::string> couples;
  std::map<std::string, bool> flag;
};
Opts parse_opts(int argc, char** argv, int start, const std::vector<std::string>& valued,
                const std::vector<std::string>& flags) {
  Opts o;
  for (int k = start; k < argc; ++k) {
    std::string a = argv[k];
    std::string v;
    const auto eq = a.find('=');
    if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    bool known = false;
    for (const auto& f : flags)
      if (a == f) {
        o.flag[f] = true;
        known = true;
      }
    for (const auto& name : valued)
      if (a == name) {
        if (eq == std::string::npos) {
          if (k + 1 >= argc) invalid(a + " needs a value");
          v = argv[++k];
        }
        if (name == "--couple") o.couples.push_back(v);
        else o.val[name] = v;
        known = true;
      }
    if (!known) invalid("unknown option '" + a + "'");
  }
  return o;
}
double num(const Opts& o, const char* k, double d) {
  auto it = o.val.find(k);
  return it == o.val.end() ? d : std::stod(it->second);
}
long long inum(const Opts& o, const char* k, long long d) {
  auto it = o.val.find(k);
  return it == o.val.end() ? d : std::stoll(it->second);
}
std::string sval(const Opts& o, const char* k, const std::string& d = "") {
  auto it = o.val.find(k);
  return it == o.val.end() ? d : it->second;
}

// ---- train (cmtf_main.cpp:113-204)
int cmd_train(const Opts& o, const Json& argv) {
  const std::string tensor_path = sval(o, "--tensor"), test_path = sval(o, "--test");
  if (tensor_path.empty()) invalid("--tensor is required");
  if (!o.val.count("--rank")) invalid("--rank is required");
  const double split = num(o, "--split", 0.0);
  if (split > 0 && !test_path.empty()) invalid("--split excludes --test");
  const std::string kernel = sval(o, "--kernel", "opt");
  if (kernel != "opt" && kernel != "naive") invalid("--kernel must be naive or opt");
  const std::string out_dir = sval(o, "--out", ".");
  make_dirs(out_dir);
  const uint64_t seed = (uint64_t)inum(o, "--seed", 0);

  Coo full = load_tensor(tensor_path);
  Coo train = full, test;
  bool have_test = false;
  if (split > 0.0) {
    uint64_t n_test = 0;
    check(cmtf_split_train_test(full.order(), full.idx.data(), full.vals.data(), full.nnz(), split,
                                seed, nullptr, nullptr, nullptr, nullptr, &n_test, 0));
    train.idx.resize((full.nnz() - n_test) * full.order());
    train.vals.resize(full.nnz() - n_test);
    test.dims = full.dims;
    test.idx.resize(n_test * full.order());
    test.vals.resize(n_test);
    check(cmtf_split_train_test(full.order(), full.idx.data(), full.vals.data(), full.nnz(), split,
                                seed, train.idx.data(), train.vals.data(), test.idx.data(),
                                test.vals.data(), &n_test, 0));
    have_test = true;
  } else if (!test_path.empty()) {
    test = load_tensor(test_path);
    have_test = true;
  }
  std::vector<Couple> cps;
  std::vector<Matrix> mats;
  for (const auto& c : o.couples) cps.push_back(parse_couple(c));
  for (const auto& c : cps) mats.push_back(load_matrix(c, train));

  const std::vector<uint32_t> ranks = parse_u32_list(sval(o, "--rank"), "--rank");
  cmtf_gpu_config cfg;
  cmtf_gpu_config_default(&cfg);
  cfg.order = (int32_t)ranks.size();
  cfg.ranks = ranks.data();
  cfg.eta0 = num(o, "--eta", 1e-3);
  cfg.mu = num(o, "--mu", 0.1);
  cfg.lambda_reg = num(o, "--lreg", 0.1);
  cfg.workers = (int32_t)inum(o, "--workers", 1);
  cfg.max_epochs = (int32_t)inum(o, "--epochs", 100);
  cfg.rel_tol = num(o, "--tol", 1e-4);
  cfg.seed = seed;
  cfg.kernel = kernel == "naive" ? CMTF_KERNEL_NAIVE : CMTF_KERNEL_OPT;
  cfg.core_structure = o.flag.count("--cp") ? 1 : 0;
  cfg.nonnegative = o.flag.count("--nonneg") ? 1 : 0;
  cfg.device = device();
  if ((int)ranks.size() != train.order())
    invalid("rank list has " + std::to_string(ranks.size()) + " entries for a tensor of order " +
            std::to_string(train.order()));
  cmtf_gpu_ctx* ctx = nullptr;
  check(cmtf_gpu_create(&cfg, &ctx));
  std::unique_ptr<cmtf_gpu_ctx, int (*)(cmtf_gpu_ctx*)> own(ctx, cmtf_gpu_destroy);
  check(cmtf_gpu_set_tensor(ctx, train.dims.data(), train.idx.data(), train.vals.data(),
                            train.nnz()),
        ctx);
  for (const auto& m : mats)
    check(cmtf_gpu_add_matrix(ctx, m.mode0, m.rows, m.cols, m.idx.data(), m.vals.data(),
                              m.vals.size(), m.weight),
          ctx);
  check(cmtf_gpu_make_state(ctx), ctx);
  std::vector<double> log(4 * (size_t)std::max(1, cfg.max_epochs));
  int32_t n_log = 0;
  check(cmtf_gpu_train(ctx, log.data(), std::max(1, cfg.max_epochs), &n_log), ctx);
  double test_rmse = 0.0;
  if (have_test && test.nnz())
    check(cmtf_gpu_test_rmse(ctx, test.idx.data(), test.vals.data(), test.nnz(), &test_rmse), ctx);

  // train()'s finalised model -> model.txt (save_model, src/model_io.cpp:94-126)
  size_t core_n = 1;
  for (uint32_t j : ranks) core_n *= j;
  const bool cp_out = cfg.core_structure == 1 && cfg.nonnegative;  // the projection keeps CP
  std::vector<double> core(core_n);
  std::vector<std::vector<double>> F(ranks.size()), V(mats.size());
  std::vector<double*> fp, vp;
  std::vector<uint32_t> frows;
  for (size_t n = 0; n < ranks.size(); ++n) {
    F[n].resize((size_t)train.dims[n] * ranks[n]);
    fp.push_back(F[n].data());
    frows.push_back(train.dims[n]);
  }
  std::vector<int32_t> cmodes;
  std::vector<uint32_t> crows;
  for (size_t m = 0; m < mats.size(); ++m) {
    V[m].resize((size_t)mats[m].cols * ranks[mats[m].mode0]);
    vp.push_back(V[m].data());
    cmodes.push_back(mats[m].mode0);
    crows.push_back(mats[m].cols);
  }
  check(cmtf_gpu_finalize_model(ctx, core.data(), fp.data(), vp.empty() ? nullptr : vp.data()),
        ctx);
  const std::string model_path = out_dir + "/model.txt", log_path = out_dir + "/log.csv";
  std::vector<const double*> cfp(fp.begin(), fp.end()), cvp(vp.begin(), vp.end());
  check(cmtf_model_save(model_path.c_str(), (int32_t)ranks.size(), ranks.data(), cp_out,
                        core.data(), frows.data(), cfp.data(), (int32_t)mats.size(),
                        cmodes.data(), crows.data(), cvp.empty() ? nullptr : cvp.data()));
  // log.csv (write_log_csv, src/trainer.cpp:20-28)
  std::string csv = "epoch,train_rmse,objective,seconds\n";
  for (int e = 0; e < n_log; ++e) {
    char line[160];
    std::snprintf(line, sizeof line, "%d,%.17g,%.17g,%.6f\n", (int)log[4 * e], log[4 * e + 1],
                  log[4 * e + 2], log[4 * e + 3]);
    csv += line;
  }
  write_text(log_path, csv);
  std::string test_out;
  if (split > 0.0) {
    test_out = out_dir + "/test.tns";
    check(cmtf_coo_write(test_out.c_str(), test.order(), test.dims.data(), test.idx.data(),
                         test.vals.data(), test.nnz(), 0));
  }
  Json man = Json::object();
  man["command"] = Json::str("train");
  man["argv"] = argv;
  man["version"] = Json::str(kVersion);
  man["seed"] = Json::integer((long long)seed);
  man["inputs"]["tensor"] = Json::str(tensor_path);
  man["inputs"]["test"] = Json::str(test_path);
  man["inputs"]["split"] = Json::num(split);
  Json cj = Json::array();
  for (const auto& c : cps) {
    Json e = Json::object();
    e["mode"] = Json::integer(c.mode);
    e["path"] = Json::str(c.path);
    e["lambda"] = Json::num(c.lambda);
    cj.arr.push_back(e);
  }
  man["inputs"]["couples"] = cj;
  Json rj = Json::array();
  for (uint32_t j : ranks) rj.arr.push_back(Json::integer(j));
  man["config"]["ranks"] = rj;
  man["config"]["eta0"] = Json::num(cfg.eta0);
  man["config"]["mu"] = Json::num(cfg.mu);
  man["config"]["lambda_reg"] = Json::num(cfg.lambda_reg);
  man["config"]["workers"] = Json::integer(cfg.workers);
  man["config"]["max_epochs"] = Json::integer(cfg.max_epochs);
  man["config"]["rel_tol"] = Json::num(cfg.rel_tol);
  man["config"]["kernel"] = Json::str(kernel);
  man["config"]["cp"] = Json::boolean(cfg.core_structure == 1);
  man["config"]["nonnegative"] = Json::boolean(cfg.nonnegative);
  man["config"]["device"] = Json::str("B200 (cuda:" + std::to_string(cfg.device) + ")");
  man["outputs"]["model"] = Json::str(model_path);
  man["outputs"]["log"] = Json::str(log_path);
  if (!test_out.empty()) man["outputs"]["test_split"] = Json::str(test_out);
  std::string mtxt;
  man.dump(mtxt, 0);
  write_text(out_dir + "/manifest.json", mtxt + "\n");

  if (n_log > 0)
    std::printf("epochs=%d train_rmse=%.6g\n", (int)log[4 * (n_log - 1)], log[4 * (n_log - 1) + 1]);
  if (have_test) std::printf("test_rmse=%.6g\n", test_rmse);
  std::printf("model=%s\n", model_path.c_str());
  return 0;
}

// ---- eval (cmtf_main.cpp:215-239)
int cmd_eval(const Opts& o) {
  const std::string model_path = sval(o, "--model"), test_path = sval(o, "--test");
  if (model_path.empty()) invalid("--model is required");
  if (test_path.empty()) invalid("--test is required");
  cmtf_model_file* mf = nullptr;
  check(cmtf_model_load(model_path.c_str(), &mf));
  std::unique_ptr<cmtf_model_file, void (*)(cmtf_model_file*)> own_m(mf, cmtf_model_free);
  Coo test = load_tensor(test_path);
  std::vector<Couple> cps;
  std::vector<Matrix> mats;
  for (const auto& c : o.couples) cps.push_back(parse_couple(c));
  for (const auto& c : cps) mats.push_back(load_matrix(c, test));
  const int order = cmtf_model_order(mf);
  std::vector<uint32_t> ranks(cmtf_model_ranks(mf), cmtf_model_ranks(mf) + order);
  if (order != test.order())
    invalid("model has " + std::to_string(order) + " factors for a core of order " +
            std::to_string(test.order()));
  if (mats.size() > (size_t)cmtf_model_n_coupled(mf))
    invalid("no coupled factor for this matrix");
  cmtf_gpu_config cfg;
  cmtf_gpu_config_default(&cfg);
  cfg.order = order;
  cfg.ranks = ranks.data();
  cfg.nonnegative = 1;  // evaluation only: no orthogonalisation shape checks
  cfg.device = device();
  cmtf_gpu_ctx* ctx = nullptr;
  check(cmtf_gpu_create(&cfg, &ctx));
  std::unique_ptr<cmtf_gpu_ctx, int (*)(cmtf_gpu_ctx*)> own(ctx, cmtf_gpu_destroy);
  if (test.nnz() == 0) invalid("cannot evaluate an empty tensor");
  for (int n = 0; n < order; ++n)
    if (cmtf_model_factor_rows(mf, n) != test.dims[n])
      invalid("factor " + std::to_string(n + 1) + " has " +
              std::to_string(cmtf_model_factor_rows(mf, n)) + " rows but mode " +
              std::to_string(n + 1) + " has size " + std::to_string(test.dims[n]));
  check(cmtf_gpu_set_tensor(ctx, test.dims.data(), test.idx.data(), test.vals.data(), test.nnz()),
        ctx);
  for (const auto& m : mats)
    check(cmtf_gpu_add_matrix(ctx, m.mode0, m.rows, m.cols, m.idx.data(), m.vals.data(),
                              m.vals.size(), m.weight),
          ctx);
  std::vector<const double*> fp, vp;
  for (int n = 0; n < order; ++n) fp.push_back(cmtf_model_factor(mf, n));
  for (size_t m = 0; m < mats.size(); ++m) {
    if (cmtf_model_coupled_rows(mf, (int)m) != mats[m].cols)
      invalid("coupled factor " + std::to_string(m + 1) + " does not match its matrix");
    vp.push_back(cmtf_model_coupled(mf, (int)m));
  }
  check(cmtf_gpu_set_model(ctx, cmtf_model_core(mf), fp.data(), vp.empty() ? nullptr : vp.data()),
        ctx);
  double rmse = 0.0, obj = 0.0;
  check(cmtf_gpu_epoch_stats(ctx, 0.0, &rmse, &obj), ctx);
  std::vector<double> mr(mats.size());
  for (size_t m = 0; m < mats.size(); ++m) check(cmtf_gpu_matrix_rmse(ctx, (int)m, &mr[m]), ctx);
  if (o.flag.count("--json")) {
    Json j = Json::object();
    j["test_rmse"] = Json::num(rmse);
    j["n_entries"] = Json::integer((long long)test.nnz());
    Json a = Json::array();
    for (double v : mr) a.arr.push_back(Json::num(v));
    j["matrix_rmse"] = a;
    std::string t;
    j.dump(t, 0);
    std::printf("%s\n", t.c_str());
    return 0;
  }
  std::printf("test_rmse=%.17g\n", rmse);
  std::printf("n_entries=%llu\n", (unsigned long long)test.nnz());
  for (size_t m = 0; m < mr.size(); ++m) std::printf("matrix_rmse_%zu=%.17g\n", m + 1, mr[m]);
  return 0;
}

void usage() {
  std::fprintf(stderr,
               "usage: cmtf_b200 train --tensor PATH --rank J1,J2,... [options]\n"
               "       cmtf_b200 eval --model PATH --test PATH [--couple MODE:PATH:LAMBDA] "
               "[--json]\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 1;
  }
  const std::string sub = argv[1];
  try {
    if (sub == "train") {
      Opts o = parse_opts(argc, argv, 2,
                          {"--tensor", "--test", "--split", "--rank", "--couple", "--kernel",
                           "--eta", "--mu", "--lreg", "--workers", "--epochs", "--tol", "--seed",
                           "--out"},
                          {"--cp", "--nonneg"});
      return cmd_train(o, argv_json(argc, argv));
    }
    if (sub == "eval") {
      Opts o = parse_opts(argc, argv, 2, {"--model", "--test", "--couple"}, {"--json"});
      return cmd_eval(o);
    }
    if (sub == "--help" || sub == "-h") {
      usage();
      return 0;
    }
    usage();
    return 1;
  } catch (const Failure& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return e.code == CMTF_EDIVERGENCE ? 2 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}

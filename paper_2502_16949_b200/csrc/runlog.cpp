// Run artifacts of the reference CLI's `kge train` (tools/kge.cpp:181-247):
// train_log.jsonl (one JSON record per epoch, flushed per line), loss.log
// ("<epoch> <loss %.17g>") and summary.json, written by the engine's C ABI so
// a caller driving skg_fit / skg_train_epoch leaves the same files the
// reference does. JSON follows nlohmann::json's output: object keys sorted
// (std::map), compact dump() for the JSONL records, dump(2) for the summary,
// doubles as the shortest round-trip decimal ("1.0" for integral values).
// Host code only.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <variant>
#include <vector>

#include "../../include/skge_b200.h"

namespace {

thread_local std::string g_log_err;

// Shortest decimal that reads back as the same double, in the style of
// nlohmann::json / Python repr: positional for exponents in [-4, 15], else
// d.ddde+XX.
std::string fmt_double(double v) {
  if (std::isnan(v) || std::isinf(v)) return "null";  // nlohmann writes non-finite numbers as null
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  // buf = [-]d.ddde[+-]XX with prec significant digits
  std::string s(buf);
  const bool neg = s[0] == '-';
  if (neg) s.erase(0, 1);
  const size_t epos = s.find('e');
  const int exp10 = std::atoi(s.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits += s[i];
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  std::string out;
  const int nd = static_cast<int>(digits.size());
  if (exp10 >= -4 && exp10 < 16) {
    if (exp10 >= 0) {
      if (nd <= exp10 + 1) {
        out = digits + std::string(static_cast<size_t>(exp10 + 1 - nd), '0') + ".0";
      } else {
        out = digits.substr(0, static_cast<size_t>(exp10 + 1)) + "." + digits.substr(static_cast<size_t>(exp10 + 1));
      }
    } else {
      out = "0." + std::string(static_cast<size_t>(-exp10 - 1), '0') + digits;
    }
  } else {
    out = digits.substr(0, 1);
    if (nd > 1) out += "." + digits.substr(1);
    char e[16];
    std::snprintf(e, sizeof e, "e%c%02d", exp10 < 0 ? '-' : '+', std::abs(exp10));
    out += e;
  }
  return neg ? "-" + out : out;
}

std::string quote(const std::string& s) {
  std::string o = "\"";
  for (const unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      case '\r': o += "\\r"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += static_cast<char>(c);
        }
    }
  }
  return o + "\"";
}

// Minimal JSON value with nlohmann's output conventions.
struct J {
  enum Kind { Null, Int, UInt, Dbl, Str, Obj } kind = Null;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0;
  std::string s;
  std::map<std::string, J> o;  // sorted keys, like nlohmann::json's std::map objects
  static J null() { return J{}; }
  static J integer(int64_t v) {
    J j;
    j.kind = Int;
    j.i = v;
    return j;
  }
  static J uinteger(uint64_t v) {
    J j;
    j.kind = UInt;
    j.u = v;
    return j;
  }
  static J number(double v) {
    J j;
    j.kind = Dbl;
    j.d = v;
    return j;
  }
  static J string(std::string v) {
    J j;
    j.kind = Str;
    j.s = std::move(v);
    return j;
  }
  static J object() {
    J j;
    j.kind = Obj;
    return j;
  }
  J& operator[](const std::string& k) { return o[k]; }
  void dump(std::string& out, int indent, int level) const {
    switch (kind) {
      case Null: out += "null"; return;
      case Int: out += std::to_string(i); return;
      case UInt: out += std::to_string(u); return;
      case Dbl: out += fmt_double(d); return;
      case Str: out += quote(s); return;
      case Obj: break;
    }
    if (o.empty()) {
      out += "{}";
      return;
    }
    out += "{";
    bool first = true;
    for (const auto& kv : o) {
      if (!first) out += ",";
      first = false;
      if (indent >= 0) out += "\n" + std::string(static_cast<size_t>(indent * (level + 1)), ' ');
      out += quote(kv.first) + (indent >= 0 ? ": " : ":");
      kv.second.dump(out, indent, level + 1);
    }
    if (indent >= 0) out += "\n" + std::string(static_cast<size_t>(indent * level), ' ');
    out += "}";
  }
  std::string dump(int indent = -1) const {
    std::string out;
    dump(out, indent, 0);
    return out;
  }
};

const char* model_name(uint32_t m) {  // common.hpp:82-93
  static const char* n[] = {"transe", "transr", "transh", "toruse", "distmult", "complex", "rotate"};
  return m < 7 ? n[m] : "unknown";
}

// kge.cpp:146-160
double flops_per_epoch(const skg_model_config& mc, int64_t m) {
  const double M = double(m), de = double(mc.dim_entity), dr = double(mc.dim_relation);
  const double spmm = 4.0 * 3.0 * M * dr;
  const double norms = 4.0 * 3.0 * M * dr;
  double extra = 0.0;
  switch (mc.model) {
    case SKG_TRANSR: extra = 8.0 * M * de * dr; break;
    case SKG_TRANSH: extra = 12.0 * M * de; break;
    case SKG_DISTMULT: extra = 4.0 * M * dr; break;
    case SKG_COMPLEX:
    case SKG_ROTATE: extra = 16.0 * M * dr; break;
    default: break;
  }
  return spmm + norms + extra;
}

}  // namespace

struct skg_run_log {
  std::string dir, log_path, loss_path;
  std::ofstream log, loss;
};

extern "C" {

const char* skg_run_log_last_error(void) { return g_log_err.c_str(); }

skg_status skg_run_log_open(const char* out_dir, skg_run_log** out) {
  if (!out || !out_dir) return SKG_ERR_CONFIG;
  *out = nullptr;
  try {
    auto lg = std::make_unique<skg_run_log>();
    lg->dir = out_dir;
    std::filesystem::create_directories(lg->dir);
    lg->log_path = lg->dir + "/train_log.jsonl";
    lg->loss_path = lg->dir + "/loss.log";
    lg->log.open(lg->log_path, std::ios::app);
    lg->loss.open(lg->loss_path, std::ios::app);
    if (!lg->log || !lg->loss) {  // kge.cpp:191-194
      g_log_err = "cannot open log files under " + lg->dir;
      return SKG_ERR_PARSE;
    }
    *out = lg.release();
    return SKG_OK;
  } catch (const std::exception& e) {
    g_log_err = e.what();
    return SKG_ERR_PARSE;
  }
}

// kge.cpp:198-208: one compact JSON record per epoch, flushed (a crashed run
// still leaves whole, parseable lines), and "<epoch> <loss %.17g>".
skg_status skg_run_log_epoch(skg_run_log* lg, const skg_epoch_report* r) {
  if (!lg || !r) return SKG_ERR_CONFIG;
  J j = J::object();
  j["epoch"] = J::integer(r->epoch);
  j["loss"] = J::number(static_cast<double>(static_cast<float>(r->loss)));  // Real loss, stored as double
  j["t_forward_s"] = J::number(r->t_forward_s);
  j["t_backward_s"] = J::number(r->t_backward_s);
  j["t_step_s"] = J::number(r->t_step_s);
  lg->log << j.dump() << "\n";
  lg->log.flush();
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", static_cast<double>(static_cast<float>(r->loss)));
  lg->loss << r->epoch << " " << buf << "\n";
  lg->loss.flush();
  if (!lg->log || !lg->loss) {
    g_log_err = "write failed under " + lg->dir;
    return SKG_ERR_PARSE;
  }
  return SKG_OK;
}

// kge.cpp:210-240: summary.json of the run (dump(2), sorted keys).
skg_status skg_run_log_summary(skg_run_log* lg, const skg_model_config* mc, const skg_train_config* tc,
                               const skg_run_summary* info) {
  if (!lg || !mc || !tc || !info) return SKG_ERR_CONFIG;
  try {
    J s = J::object();
    s["model"] = J::string(model_name(mc->model));
    s["norm"] = J::string(mc->norm == SKG_L1 ? "l1" : "l2");
    s["dim_entity"] = J::integer(mc->dim_entity);
    s["dim_relation"] = J::integer(mc->dim_relation);
    s["engine"] = J::string(info->engine ? info->engine : "sparse");
    J ds = J::object();
    ds["source"] = J::string(info->dataset_source ? info->dataset_source : "synthetic");
    ds["entities"] = J::integer(info->entities);
    ds["relations"] = J::integer(info->relations);
    ds["train"] = J::integer(info->train);
    ds["valid"] = J::integer(info->valid);
    ds["test"] = J::integer(info->test);
    ds["dropped_valid"] = J::integer(info->dropped_valid);
    ds["dropped_test"] = J::integer(info->dropped_test);
    s["dataset"] = ds;
    J cfg = J::object();
    cfg["lr"] = J::number(static_cast<double>(tc->lr));
    cfg["margin"] = J::number(static_cast<double>(tc->margin));
    cfg["epochs"] = J::integer(tc->epochs);
    cfg["batch_size"] = J::integer(tc->batch_size);
    cfg["seed"] = J::uinteger(tc->seed);
    cfg["threads"] = J::integer(info->threads);
    if (tc->has_scheduler) {
      J sch = J::object();
      sch["every_epochs"] = J::integer(tc->decay_every);
      sch["factor"] = J::number(static_cast<double>(tc->decay_factor));
      cfg["scheduler"] = sch;
    } else {
      cfg["scheduler"] = J::null();
    }
    s["config"] = cfg;
    s["final_loss"] = info->epochs_run > 0 ? J::number(static_cast<double>(static_cast<float>(info->final_loss)))
                                           : J::null();
    J tm = J::object();
    tm["forward_s"] = J::number(info->t_forward_s);
    tm["backward_s"] = J::number(info->t_backward_s);
    tm["step_s"] = J::number(info->t_step_s);
    tm["total_s"] = J::number(info->t_forward_s + info->t_backward_s + info->t_step_s);
    s["time"] = tm;
    J fl = J::object();
    const double fpe = flops_per_epoch(*mc, info->train);
    fl["per_epoch_estimate"] = J::number(fpe);
    fl["total_estimate"] = J::number(fpe * double(tc->epochs));
    s["flops"] = fl;
    J art = J::object();
    art["checkpoint"] = J::string(info->checkpoint_path ? info->checkpoint_path : (lg->dir + "/checkpoint.bin"));
    art["log"] = J::string(lg->log_path);
    art["loss_log"] = J::string(lg->loss_path);
    s["artifacts"] = art;
    std::ofstream f(lg->dir + "/summary.json");
    f << s.dump(2) << "\n";
    if (!f) {
      g_log_err = "cannot write " + lg->dir + "/summary.json";
      return SKG_ERR_PARSE;
    }
    return SKG_OK;
  } catch (const std::exception& e) {
    g_log_err = e.what();
    return SKG_ERR_PARSE;
  }
}

void skg_run_log_close(skg_run_log* lg) { delete lg; }

}  // extern "C"

// Minimal CLI11 subset — TEST INFRASTRUCTURE ONLY (oracle/).
//
// The reference's command-line front end (proj/tools/graspmatch_cli.cpp)
// includes <CLI11.hpp>, which the reference vendors under proj/vendor/ (not
// present here, proj/.gitignore:2).  This header implements exactly the part
// of CLI11's interface that file uses — App with subcommands, add_option for
// strings / numbers / std::optional / std::vector, required(),
// check(CLI::PositiveNumber), expected(n), parsed() and CLI11_PARSE — so the
// reference CLI compiles unmodified (oracle/Makefile `cli`).  Builder-written,
// not CLI11 source.
#pragma once

#include <cstdio>
#include <functional>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("help", 0) {}
};

// A validator: returns an error message ("" = accepted).
struct Validator {
  std::function<std::string(const std::string&)> fn;
};
inline const Validator PositiveNumber{[](const std::string& s) -> std::string {
  try {
    size_t used = 0;
    const double v = std::stod(s, &used);
    if (used == s.size() && v > 0.0) return "";
  } catch (...) {
  }
  return "Value " + s + " not a positive number";
}};

namespace detail {
template <typename T>
struct is_optional : std::false_type {};
template <typename T>
struct is_optional<std::optional<T>> : std::true_type {};
template <typename T>
struct is_vector : std::false_type {};
template <typename T>
struct is_vector<std::vector<T>> : std::true_type {};

template <typename T>
T convert(const std::string& s, const std::string& name) {
  std::istringstream in(s);
  T v{};
  in >> v;
  if (in.fail() || !in.eof()) throw ParseError("Could not convert: " + name + " = " + s, 106);
  return v;
}
template <>
inline std::string convert<std::string>(const std::string& s, const std::string&) {
  return s;
}
}  // namespace detail

class Option {
 public:
  std::vector<std::string> names;  // "-c", "--config"
  std::string desc;
  bool is_required = false, seen = false;
  int n_expected = 1;
  std::vector<Validator> checks;
  std::function<void(const std::vector<std::string>&)> assign;

  Option* required() {
    is_required = true;
    return this;
  }
  Option* check(const Validator& v) {
    checks.push_back(v);
    return this;
  }
  Option* expected(int n) {
    n_expected = n;
    return this;
  }
  bool matches(const std::string& tok) const {
    for (const auto& n : names)
      if (n == tok) return true;
    return false;
  }
};

class App {
 public:
  explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)),
                                                                       name_(std::move(name)) {}

  App* require_subcommand(int n) {
    require_sub_ = n;
    return this;
  }

  App* add_subcommand(const std::string& name, const std::string& description) {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }

  template <typename T>
  Option* add_option(const std::string& spec, T& var, const std::string& description) {
    auto opt = std::make_unique<Option>();
    std::string s = spec, part;
    std::istringstream in(s);
    while (std::getline(in, part, ','))
      if (!part.empty()) opt->names.push_back(part);
    opt->desc = description;
    const std::string label = opt->names.back();
    if constexpr (detail::is_vector<T>::value) {
      opt->assign = [&var, label](const std::vector<std::string>& vals) {
        var.clear();
        for (const auto& v : vals) var.push_back(detail::convert<typename T::value_type>(v, label));
      };
    } else if constexpr (detail::is_optional<T>::value) {
      opt->assign = [&var, label](const std::vector<std::string>& vals) {
        var = detail::convert<typename T::value_type>(vals.at(0), label);
      };
    } else {
      opt->assign = [&var, label](const std::vector<std::string>& vals) {
        var = detail::convert<T>(vals.at(0), label);
      };
    }
    opts_.push_back(std::move(opt));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    size_t i = 0;
    parse_into(args, i);
  }

  int exit(const ParseError& e) const {
    if (e.code == 0) {
      std::printf("%s\n", help().c_str());
      return 0;
    }
    std::fprintf(stderr, "%s\n", e.what());
    return e.code;
  }

 private:
  std::string help() const {
    std::string h = desc_ + "\n";
    for (const auto& s : subs_) h += "  " + s->name_ + "  " + s->desc_ + "\n";
    for (const auto& o : opts_) h += "  " + o->names.back() + "  " + o->desc + "\n";
    return h;
  }

  void parse_into(const std::vector<std::string>& args, size_t& i) {
    parsed_ = true;
    int n_subs = 0;
    while (i < args.size()) {
      const std::string tok = args[i];
      if (tok == "-h" || tok == "--help") throw CallForHelp();
      App* sub = nullptr;
      for (const auto& s : subs_)
        if (s->name_ == tok) sub = s.get();
      if (sub) {
        ++i;
        ++n_subs;
        sub->parse_into(args, i);
        continue;
      }
      std::string key = tok, inline_val;
      const size_t eq = tok.find('=');
      const bool has_inline = tok.rfind("--", 0) == 0 && eq != std::string::npos;
      if (has_inline) {
        key = tok.substr(0, eq);
        inline_val = tok.substr(eq + 1);
      }
      Option* opt = nullptr;
      for (const auto& o : opts_)
        if (o->matches(key)) opt = o.get();
      if (!opt) throw ParseError("The following argument was not expected: " + tok, 109);
      std::vector<std::string> vals;
      ++i;
      if (has_inline) vals.push_back(inline_val);
      while (static_cast<int>(vals.size()) < opt->n_expected) {
        if (i >= args.size()) throw ParseError(key + ": " + std::to_string(opt->n_expected) + " required", 107);
        vals.push_back(args[i++]);
      }
      for (const auto& v : vals)
        for (const auto& c : opt->checks) {
          const std::string msg = c.fn(v);
          if (!msg.empty()) throw ParseError(key + ": " + msg, 105);
        }
      opt->assign(vals);
      opt->seen = true;
    }
    for (const auto& o : opts_)
      if (o->is_required && !o->seen) throw ParseError(o->names.back() + " is required", 106);
    if (require_sub_ > 0 && n_subs < require_sub_) throw ParseError("A subcommand is required", 106);
  }

  std::string desc_, name_;
  int require_sub_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv) \
  try {                              \
    (app).parse((argc), (argv));     \
  } catch (const CLI::ParseError& e) { \
    return (app).exit(e);            \
  }

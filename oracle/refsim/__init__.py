"""Restatement of the reference simulator ``tokensim`` (TEST ORACLE)."""
